"""Micro-benchmark: H2D of RRC-like crop boxes from pinned host images, copy engine
(cudaMemcpy2DAsync per box) vs one contiguous copy, to judge whether the DMA engines beat
the K0 zero-copy gather (~46 GB/s) on strided boxes."""
import time, numpy as np, torch
from cuda.bindings import runtime as rt
torch.cuda.init()
rng = np.random.default_rng(1)
n = 256
imgs, boxes = [], []
for i in range(n):
    H, W = int(rng.integers(256, 513)), int(rng.integers(256, 513))
    t = torch.empty(H * W * 3, dtype=torch.uint8).pin_memory()
    imgs.append((t, H, W))
    s = rng.uniform(0.08, 1.0); r = np.exp(rng.uniform(np.log(3/4), np.log(4/3)))
    bw = int(min(W, round(np.sqrt(s * H * W * r)))); bh = int(min(H, round(np.sqrt(s * H * W / r))))
    x0 = int(rng.integers(0, W - bw + 1)); y0 = int(rng.integers(0, H - bh + 1))
    boxes.append((x0, y0, bw, bh))
tot = sum(3 * b[2] * b[3] for b in boxes)
dst = torch.empty(tot + 4096, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
def run(nst):
    off = 0
    for i, ((t, H, W), (x0, y0, bw, bh)) in enumerate(zip(imgs, boxes)):
        st = streams[i % nst]
        src = t.data_ptr() + (y0 * W + x0) * 3
        e, = rt.cudaMemcpy2DAsync(dst.data_ptr() + off, bw * 3, src, W * 3, bw * 3, bh,
                                  rt.cudaMemcpyKind.cudaMemcpyHostToDevice, st.cuda_stream)
        assert e == rt.cudaError_t.cudaSuccess, e
        off += 3 * bw * bh
for nst in (1, 2, 4):
    for _ in range(3): run(nst)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); reps = 20
    for _ in range(reps): run(nst)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"memcpy2D streams={nst}: {tot/1e6:.1f} MB in {dt*1e3:.3f} ms = {tot/dt/1e9:.1f} GB/s")
big = torch.empty(tot, dtype=torch.uint8).pin_memory()
for _ in range(3): dst[:tot].copy_(big, non_blocking=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(20): dst[:tot].copy_(big, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 20
print(f"contiguous: {tot/dt/1e9:.1f} GB/s")
# CPU cost of issuing the 256 calls
t0 = time.perf_counter(); run(1); t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"issue cost per box: {(t1-t0)/n*1e6:.2f} us")
