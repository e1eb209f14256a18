/*
 * lf_oracle.c -- CPU restatement of the MinatoLoader transform chains (fp64).
 * TEST INFRASTRUCTURE ONLY: see lf_oracle.h for provenance and parity status.
 *
 * Written for clarity, not speed: straight scalar loops in the same order the
 * transforms appear in the reference chains (proj/src/workloads.cpp:103-156).
 */
#include "lf_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* mt19937_64 (Matsumoto & Nishimura 2000; the parameters std::mt19937_64
 * uses).  Restated here independently of libstdc++ so the oracle does not
 * share code with the product, which calls std::mt19937_64 directly. */
#define MT_NN 312
#define MT_MM 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void lfo_mt64_seed(lfo_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_NN; i++) {
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    g->idx = MT_NN;
}

uint64_t lfo_mt64_next(lfo_mt64* g) {
    if (g->idx >= MT_NN) {
        for (int i = 0; i < MT_NN; i++) {
            uint64_t x = (g->mt[i] & MT_UM) | (g->mt[(i + 1) % MT_NN] & MT_LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= MT_MATRIX_A;
            g->mt[i] = g->mt[(i + MT_MM) % MT_NN] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

void lfo_sample_rng(lfo_mt64* g, uint64_t seed, uint64_t id) {
    /* experiment.cpp:163 mixing constant, keyed by sample id instead of worker slot */
    lfo_mt64_seed(g, seed ^ (0x9e3779b97f4a7c15ULL * (id + 1ULL)));
}

double lfo_unif01(lfo_mt64* g) { return (double)(lfo_mt64_next(g) >> 11) * 0x1.0p-53; }

int64_t lfo_randint(lfo_mt64* g, int64_t lo, int64_t hi) {
    double u = lfo_unif01(g);
    int64_t span = hi - lo + 1;
    int64_t k = (int64_t)floor(u * (double)span);
    if (k >= span) k = span - 1;
    return lo + k;
}

double lfo_uniform(lfo_mt64* g, double a, double b) { return a + (b - a) * lfo_unif01(g); }

/* ------------------------------------------------------------------ */
/* Philox4x32-10 */
static void mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    *lo = (uint32_t)p;
}

void lfo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo32(0xD2511F53u, c0, &hi0, &lo0);
        mulhilo32(0xCD9E8D57u, c2, &hi1, &lo1);
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Box-Muller on a pair of 32-bit uniforms: u = (x + 0.5) * 2^-32 in (0,1). */
static void box_muller(uint32_t xa, uint32_t xb, double* z0, double* z1) {
    const double two_m32 = 0x1.0p-32;
    double u1 = ((double)xa + 0.5) * two_m32;
    double u2 = ((double)xb + 0.5) * two_m32;
    double r = sqrt(-2.0 * log(u1));
    double th = 2.0 * M_PI * u2;
    *z0 = r * cos(th);
    *z1 = r * sin(th);
}

void lfo_normals4(uint64_t group, uint32_t k0, uint32_t k1, double z[4]) {
    uint32_t ctr[4] = {(uint32_t)group, (uint32_t)(group >> 32), 0u, 0u};
    uint32_t key[2] = {k0, k1};
    uint32_t r[4];
    lfo_philox4x32_10(ctr, key, r);
    box_muller(r[0], r[1], &z[0], &z[1]);
    box_muller(r[2], r[3], &z[2], &z[3]);
}

/* ------------------------------------------------------------------ */
/* img_seg chain: RandomCrop, RandomFlip, RandomBrightness, GaussianNoise, Cast
 * (proj/src/workloads.cpp:142-148), plus the optional RandomZoom3D (trilinear
 * resample of a zoomed window) and RandomContrast ops.  Parameter draws: see
 * lfo_draw3d (11 draws for the reference chain; the stream position never
 * depends on outcomes).
 * Output voxel v = (z*ch + y)*cw + x reads input
 *   (off_d + (flip_d ? cd-1-z : z), off_h + ..., off_w + ...), zero outside;
 *   img_out = img_in * scale + sigma * N_v, lbl_out = lbl_in,
 * N_v = normal (v & 3) of Philox group v >> 2 (lfo_normals4).           */

void lfo_cfg3d_default(lfo_cfg3d* c) {
    c->crop[0] = c->crop[1] = c->crop[2] = 128;
    c->p_flip = 1.0 / 3.0;
    c->p_bright = 0.1;
    c->bright_lo = 0.7;
    c->bright_hi = 1.3;
    c->p_noise = 0.1;
    c->noise_std_max = 0.1;
    c->has_zoom = 0;
    c->p_zoom = 0.5;
    c->zoom_lo = 0.8;
    c->zoom_hi = 1.2;
    c->has_contrast = 0;
    c->p_contrast = 0.15;
    c->contrast_lo = 0.75;
    c->contrast_hi = 1.25;
    c->has_fg = 0;
    c->p_fg = 0.4;
}

/* Draw order, in chain order: RandomCrop u_off[3] (the offset uniforms; the
 * offset is floor(u * (room + 1)) once the window edge is known, which equals
 * randint(0, room) of the plain chain); [RandomZoom3D: apply, factor];
 * RandomFlip x3; RandomBrightness apply, factor; [RandomContrast: apply,
 * factor]; GaussianNoise apply, std; Philox key.  Bracketed draws happen only
 * when the op is in the chain. */
void lfo_draw3d(const lfo_cfg3d* c, uint64_t seed, uint64_t id, const int64_t dims[3],
                lfo_params3d* p) {
    lfo_mt64 g;
    lfo_sample_rng(&g, seed, id);
    double u_off[3];
    for (int a = 0; a < 3; a++) u_off[a] = lfo_unif01(&g);
    p->fg = 0;
    p->u_cls = 0.0;
    p->u_adj[0] = p->u_adj[1] = p->u_adj[2] = 0.0;
    if (c->has_fg) {   /* RandomCrop's foreground draws */
        p->fg = lfo_unif01(&g) < c->p_fg;
        p->u_cls = lfo_unif01(&g);
        for (int a = 0; a < 3; a++) p->u_adj[a] = lfo_unif01(&g);
    }
    for (int a = 0; a < 3; a++) p->win[a] = c->crop[a];
    if (c->has_zoom) {
        int z_apply = lfo_unif01(&g) < c->p_zoom;
        double zf = lfo_uniform(&g, c->zoom_lo, c->zoom_hi);
        if (z_apply) {
            for (int a = 0; a < 3; a++) {
                int64_t w = (int64_t)floor((double)c->crop[a] * zf + 0.5);
                p->win[a] = w < 1 ? 1 : w;
            }
        }
    }
    for (int a = 0; a < 3; a++) {
        int64_t room = dims[a] - p->win[a];
        int64_t span = (room > 0 ? room : 0) + 1;
        int64_t k = (int64_t)floor(u_off[a] * (double)span);
        p->off[a] = k >= span ? span - 1 : k;
    }
    for (int a = 0; a < 3; a++) p->flip[a] = lfo_unif01(&g) < c->p_flip;
    int b_apply = lfo_unif01(&g) < c->p_bright;
    double b_factor = lfo_uniform(&g, c->bright_lo, c->bright_hi);
    p->scale = b_apply ? b_factor : 1.0;
    p->contrast = 1.0;
    if (c->has_contrast) {
        int c_apply = lfo_unif01(&g) < c->p_contrast;
        double c_factor = lfo_uniform(&g, c->contrast_lo, c->contrast_hi);
        if (c_apply) p->contrast = c_factor;
    }
    int n_apply = lfo_unif01(&g) < c->p_noise;
    double n_std = lfo_uniform(&g, 0.0, c->noise_std_max);
    uint64_t key = lfo_mt64_next(&g);
    p->sigma = n_apply ? n_std : 0.0;
    p->key[0] = (uint32_t)key;
    p->key[1] = (uint32_t)(key >> 32);
}

/* PyTorch area_pixel_compute_source_index (align_corners=False, linear) on
 * scale = in / out, then the upsample_linear tap pair and weights. */
static void linear_taps(int64_t dst, int64_t in, int64_t out, int64_t* i0, int64_t* i1, double* l0,
                        double* l1) {
    double scale = (double)in / (double)out;
    double src = scale * ((double)dst + 0.5) - 0.5;
    if (src < 0.0) src = 0.0;
    int64_t a = (int64_t)floor(src);
    if (a > in - 1) a = in - 1;
    *i0 = a;
    *i1 = a < in - 1 ? a + 1 : a;
    *l1 = src - (double)a;
    *l0 = 1.0 - *l1;
}

static double vox_or_zero(const float* img, const int64_t dims[3], int64_t z, int64_t y, int64_t x) {
    if (z >= dims[0] || y >= dims[1] || x >= dims[2]) return 0.0;
    return (double)img[(z * dims[1] + y) * dims[2] + x];
}

int lfo_fg_offsets(const lfo_params3d* p, const uint8_t* lbl, const int64_t dims[3], int64_t off[3]) {
    if (!p->fg) return -1;
    int64_t lo[8][3], hi[8][3];
    int present[8] = {0};
    for (int k = 0; k < 8; k++)
        for (int a = 0; a < 3; a++) {
            lo[k][a] = INT64_MAX;
            hi[k][a] = -1;
        }
    for (int64_t z = 0; z < dims[0]; z++)
        for (int64_t y = 0; y < dims[1]; y++)
            for (int64_t x = 0; x < dims[2]; x++) {
                const int v = lbl[(z * dims[1] + y) * dims[2] + x];
                if (v < 1 || v > 7) continue;
                const int64_t q[3] = {z, y, x};
                present[v] = 1;
                for (int a = 0; a < 3; a++) {
                    if (q[a] < lo[v][a]) lo[v][a] = q[a];
                    if (q[a] > hi[v][a]) hi[v][a] = q[a];
                }
            }
    int cls[7], n = 0;
    for (int v = 1; v <= 7; v++)
        if (present[v]) cls[n++] = v;
    if (n == 0) return -1;
    int64_t k = (int64_t)floor(p->u_cls * (double)n);
    if (k >= n) k = n - 1;
    const int cl = cls[k];
    for (int a = 0; a < 3; a++) {
        const int64_t patch = p->win[a], l = lo[cl][a], h = hi[cl][a] + 1;
        int64_t diff = patch - (h - l);
        const int64_t sign = diff < 0 ? -1 : 1;
        if (diff < 0) diff = -diff;
        int64_t ladj = diff > 0 ? (int64_t)floor(p->u_adj[a] * (double)diff) : 0;
        if (ladj >= diff && diff > 0) ladj = diff - 1;
        const int64_t hadj = diff - ladj;
        int64_t low = l - sign * ladj, high = h + sign * hadj;
        if (low < 0) low = 0;
        if (high > dims[a]) high = dims[a];
        const int64_t d2 = patch - (high - low);
        if (d2 > 0) {
            if (low == 0) high += d2;
            else low -= d2;
        }
        const int64_t room = dims[a] - patch > 0 ? dims[a] - patch : 0;
        off[a] = low < 0 ? 0 : (low > room ? room : low);
    }
    return 0;
}

void lfo_apply3d(const lfo_cfg3d* c, const lfo_params3d* p0, const float* img,
                 const uint8_t* lbl, const int64_t dims[3], double* out_img,
                 uint8_t* out_lbl) {
    lfo_params3d fgp = *p0;   /* foreground-biased crops move the window */
    const lfo_params3d* p = p0;
    if (c->has_fg && lfo_fg_offsets(p0, lbl, dims, fgp.off) == 0) p = &fgp;
    const int64_t cd = c->crop[0], ch = c->crop[1], cw = c->crop[2];
    const int64_t D = dims[0], H = dims[1], W = dims[2];
    const int64_t* win = p->win;
    const int64_t n = cd * ch * cw;
    /* 1. RandomCrop [+ RandomZoom3D resample] + RandomFlip + RandomBrightness */
    double sum = 0.0;
    for (int64_t z = 0; z < cd; z++) {
        int64_t wz = p->flip[0] ? cd - 1 - z : z;   /* output position before the flip */
        for (int64_t y = 0; y < ch; y++) {
            int64_t wy = p->flip[1] ? ch - 1 - y : y;
            for (int64_t x = 0; x < cw; x++) {
                int64_t wx = p->flip[2] ? cw - 1 - x : x;
                int64_t v = (z * ch + y) * cw + x;
                double val = 0.0;
                uint8_t l = 0;
                if (win[0] == cd && win[1] == ch && win[2] == cw) {
                    int64_t sz = p->off[0] + wz, sy = p->off[1] + wy, sx = p->off[2] + wx;
                    if (sz < D && sy < H && sx < W) {
                        int64_t si = (sz * H + sy) * W + sx;
                        val = (double)img[si];
                        l = lbl[si];
                    }
                } else {
                    int64_t z0, z1, y0, y1, x0, x1;
                    double lz0, lz1, ly0, ly1, lx0, lx1;
                    linear_taps(wz, win[0], cd, &z0, &z1, &lz0, &lz1);
                    linear_taps(wy, win[1], ch, &y0, &y1, &ly0, &ly1);
                    linear_taps(wx, win[2], cw, &x0, &x1, &lx0, &lx1);
                    const int64_t oz = p->off[0], oy = p->off[1], ox = p->off[2];
                    val = lz0 * (ly0 * (lx0 * vox_or_zero(img, dims, oz + z0, oy + y0, ox + x0) +
                                        lx1 * vox_or_zero(img, dims, oz + z0, oy + y0, ox + x1)) +
                                 ly1 * (lx0 * vox_or_zero(img, dims, oz + z0, oy + y1, ox + x0) +
                                        lx1 * vox_or_zero(img, dims, oz + z0, oy + y1, ox + x1))) +
                          lz1 * (ly0 * (lx0 * vox_or_zero(img, dims, oz + z1, oy + y0, ox + x0) +
                                        lx1 * vox_or_zero(img, dims, oz + z1, oy + y0, ox + x1)) +
                                 ly1 * (lx0 * vox_or_zero(img, dims, oz + z1, oy + y1, ox + x0) +
                                        lx1 * vox_or_zero(img, dims, oz + z1, oy + y1, ox + x1)));
                    int64_t nz = wz * win[0] / cd, ny = wy * win[1] / ch, nx = wx * win[2] / cw;
                    if (nz > win[0] - 1) nz = win[0] - 1;
                    if (ny > win[1] - 1) ny = win[1] - 1;
                    if (nx > win[2] - 1) nx = win[2] - 1;
                    int64_t sz = oz + nz, sy = oy + ny, sx = ox + nx;
                    if (sz < D && sy < H && sx < W) l = lbl[(sz * H + sy) * W + sx];
                }
                sum += val;
                out_img[v] = val * p->scale;               /* RandomBrightness */
                out_lbl[v] = l;                            /* Cast: u8 label */
            }
        }
    }
    /* 2. RandomContrast: (v - m) * c + m, m = mean of the brightness-scaled crop */
    if (p->contrast != 1.0) {
        double m = sum / (double)n * p->scale;
        for (int64_t v = 0; v < n; v++) out_img[v] = (out_img[v] - m) * p->contrast + m;
    }
    /* 3. GaussianNoise, Cast (f32 image) */
    if (p->sigma != 0.0) {
        for (int64_t v = 0; v < n; v++) {
            double zz[4];
            lfo_normals4((uint64_t)v >> 2, p->key[0], p->key[1], zz);
            out_img[v] += p->sigma * zz[v & 3];
        }
    }
}

/* ------------------------------------------------------------------ */
/* obj_det / ImageNet chain: Resize (RandomResizedCrop), RandomHorizontalFlip,
 * ToTensor, Normalize (proj/src/workloads.cpp:151-156).  Parameter draws
 * restate torchvision RandomResizedCrop.get_params (scale, ratio, 10 tries,
 * centre-crop fallback) on the mt19937_64 primitives, then one flip draw. */

void lfo_cfg2d_default(lfo_cfg2d* c) {
    c->out_h = c->out_w = 224;
    c->scale_lo = 0.08;
    c->scale_hi = 1.0;
    c->ratio_lo = 3.0 / 4.0;
    c->ratio_hi = 4.0 / 3.0;
    c->p_hflip = 0.5;
    c->mean[0] = 0.485; c->mean[1] = 0.456; c->mean[2] = 0.406;
    c->std[0] = 0.229;  c->std[1] = 0.224;  c->std[2] = 0.225;
}

void lfo_draw2d(const lfo_cfg2d* c, uint64_t seed, uint64_t id, int64_t H, int64_t W,
                lfo_params2d* p) {
    lfo_mt64 g;
    lfo_sample_rng(&g, seed, id);
    const double area = (double)H * (double)W;
    const double lr0 = log(c->ratio_lo), lr1 = log(c->ratio_hi);
    int found = 0;
    for (int t = 0; t < 10 && !found; t++) {
        double target = area * lfo_uniform(&g, c->scale_lo, c->scale_hi);
        double aspect = exp(lfo_uniform(&g, lr0, lr1));
        int64_t w = (int64_t)nearbyint(sqrt(target * aspect)); /* round half even */
        int64_t h = (int64_t)nearbyint(sqrt(target / aspect));
        if (w > 0 && w <= W && h > 0 && h <= H) {
            p->top = lfo_randint(&g, 0, H - h);
            p->left = lfo_randint(&g, 0, W - w);
            p->h = h;
            p->w = w;
            found = 1;
        }
    }
    if (!found) {
        double in_ratio = (double)W / (double)H;
        int64_t w, h;
        if (in_ratio < c->ratio_lo) {
            w = W;
            h = (int64_t)nearbyint((double)w / c->ratio_lo);
        } else if (in_ratio > c->ratio_hi) {
            h = H;
            w = (int64_t)nearbyint((double)h * c->ratio_hi);
        } else {
            w = W;
            h = H;
        }
        p->top = (H - h) / 2;
        p->left = (W - w) / 2;
        p->h = h;
        p->w = w;
    }
    p->flip = lfo_unif01(&g) < c->p_hflip;
}

/* PyTorch upsample_bilinear2d, align_corners=False, antialias=False:
 * src = (dst + 0.5) * in/out - 0.5, clamped at 0; i0 = floor(src),
 * i1 = min(i0 + 1, in - 1), l1 = src - i0, l0 = 1 - l1. */
static void bilinear_index(int64_t dst, int64_t in, int64_t out, int64_t* i0, int64_t* i1,
                           double* l0, double* l1) {
    double scale = (double)in / (double)out;
    double src = ((double)dst + 0.5) * scale - 0.5;
    if (src < 0.0) src = 0.0;
    int64_t a = (int64_t)floor(src);
    if (a > in - 1) a = in - 1;
    *i0 = a;
    *i1 = a < in - 1 ? a + 1 : a;
    *l1 = src - (double)a;
    *l0 = 1.0 - *l1;
}

void lfo_bilinear_chw(const float* src, int64_t C, int64_t H, int64_t W, int64_t oh,
                      int64_t ow, double* out) {
    for (int64_t c = 0; c < C; c++)
        for (int64_t y = 0; y < oh; y++) {
            int64_t y0, y1; double ly0, ly1;
            bilinear_index(y, H, oh, &y0, &y1, &ly0, &ly1);
            for (int64_t x = 0; x < ow; x++) {
                int64_t x0, x1; double lx0, lx1;
                bilinear_index(x, W, ow, &x0, &x1, &lx0, &lx1);
                const float* s = src + c * H * W;
                double v = ly0 * (lx0 * s[y0 * W + x0] + lx1 * s[y0 * W + x1]) +
                           ly1 * (lx0 * s[y1 * W + x0] + lx1 * s[y1 * W + x1]);
                out[(c * oh + y) * ow + x] = v;
            }
        }
}

void lfo_apply2d(const lfo_cfg2d* c, const lfo_params2d* p, const uint8_t* src, int64_t H,
                 int64_t W, double* out) {
    const int64_t oh = c->out_h, ow = c->out_w;
    (void)H;
    for (int64_t y = 0; y < oh; y++) {
        int64_t y0, y1; double ly0, ly1;
        bilinear_index(y, p->h, oh, &y0, &y1, &ly0, &ly1);
        for (int64_t x = 0; x < ow; x++) {
            int64_t x0, x1; double lx0, lx1;
            bilinear_index(x, p->w, ow, &x0, &x1, &lx0, &lx1);
            int64_t xo = p->flip ? ow - 1 - x : x;        /* RandomHorizontalFlip */
            for (int ch = 0; ch < 3; ch++) {
#define PX(yy, xx) ((double)src[((p->top + (yy)) * W + (p->left + (xx))) * 3 + ch])
                double v = ly0 * (lx0 * PX(y0, x0) + lx1 * PX(y0, x1)) +
                           ly1 * (lx0 * PX(y1, x0) + lx1 * PX(y1, x1));
#undef PX
                double t = v / 255.0;                     /* ToTensor */
                out[(ch * oh + y) * ow + xo] = (t - c->mean[ch]) / c->std[ch]; /* Normalize */
            }
        }
    }
}

/* ------------------------------------------------------------------ */
/* speech chain: Pad, SpecAugment, FilterBank, FrameSplicing, PermuteAudio
 * (proj/src/workloads.cpp:103-111).  FilterBank = torch.stft(center=True,
 * pad_mode='reflect', window=hann(win_length, periodic) zero-padded to n_fft
 * and centred) -> |X|^2 -> slaney/slaney mel (torchaudio melscale_fbanks
 * norm='slaney', mel_scale='slaney') -> log(x + eps).  SpecAugment masks are
 * drawn at their chain position (before FilterBank, as in the reference cost
 * chain) and applied to the log-mel (mask value 0), the only representation
 * on which they are defined.  Draw order: for each freq mask w = randint(0,
 * freq_mask_max), lo = randint(0, n_mels - w); for each time mask w =
 * randint(0, floor(frac*T)), lo = randint(0, max(T - w, 0)). */

void lfo_cfgsp_default(lfo_cfgsp* c) {
    c->n_fft = 512;
    c->win_length = 320;
    c->hop = 160;
    c->n_mels = 80;
    c->sample_rate = 16000.0;
    c->f_min = 0.0;
    c->f_max = 8000.0;
    c->log_eps = 0x1.0p-24;
    c->freq_masks = 2;
    c->freq_mask_max = 27;
    c->time_masks = 10;
    c->time_mask_frac = 0.05;
}

int32_t lfo_sp_frames(const lfo_cfgsp* c, int64_t L) { return (int32_t)(1 + L / c->hop); }

void lfo_drawsp(const lfo_cfgsp* c, uint64_t seed, uint64_t id, int64_t L, lfo_paramssp* p) {
    lfo_mt64 g;
    lfo_sample_rng(&g, seed, id);
    int32_t T = lfo_sp_frames(c, L);
    p->n_frames = T;
    p->n_fmask = c->freq_masks;
    for (int i = 0; i < c->freq_masks; i++) {
        int32_t w = (int32_t)lfo_randint(&g, 0, c->freq_mask_max);
        if (w > c->n_mels) w = c->n_mels;
        p->f_w[i] = w;
        p->f_lo[i] = (int32_t)lfo_randint(&g, 0, c->n_mels - w);
    }
    p->n_tmask = c->time_masks;
    int32_t tmax = (int32_t)floor(c->time_mask_frac * (double)T);
    for (int i = 0; i < c->time_masks; i++) {
        int32_t w = (int32_t)lfo_randint(&g, 0, tmax);
        p->t_w[i] = w;
        int32_t room = T - w;
        p->t_lo[i] = (int32_t)lfo_randint(&g, 0, room > 0 ? room : 0);
    }
}

static double hz_to_mel_slaney(double f) {
    const double f_sp = 200.0 / 3.0, min_log_hz = 1000.0;
    const double min_log_mel = min_log_hz / f_sp, logstep = log(6.4) / 27.0;
    if (f >= min_log_hz) return min_log_mel + log(f / min_log_hz) / logstep;
    return f / f_sp;
}

static double mel_to_hz_slaney(double m) {
    const double f_sp = 200.0 / 3.0, min_log_hz = 1000.0;
    const double min_log_mel = min_log_hz / f_sp, logstep = log(6.4) / 27.0;
    if (m >= min_log_mel) return min_log_hz * exp(logstep * (m - min_log_mel));
    return f_sp * m;
}

void lfo_mel_fbank(const lfo_cfgsp* c, double* fb) {
    const int nf = c->n_fft / 2 + 1, nm = c->n_mels;
    double* all_freqs = (double*)malloc(sizeof(double) * nf);
    double* f_pts = (double*)malloc(sizeof(double) * (nm + 2));
    for (int k = 0; k < nf; k++) all_freqs[k] = (c->sample_rate / 2.0) * k / (nf - 1);
    double m_min = hz_to_mel_slaney(c->f_min), m_max = hz_to_mel_slaney(c->f_max);
    for (int i = 0; i < nm + 2; i++)
        f_pts[i] = mel_to_hz_slaney(m_min + (m_max - m_min) * i / (nm + 1));
    for (int m = 0; m < nm; m++) {
        double f_lo = f_pts[m], f_c = f_pts[m + 1], f_hi = f_pts[m + 2];
        double enorm = 2.0 / (f_hi - f_lo); /* slaney norm */
        for (int k = 0; k < nf; k++) {
            double down = (all_freqs[k] - f_lo) / (f_c - f_lo);
            double up = (f_hi - all_freqs[k]) / (f_hi - f_c);
            double v = down < up ? down : up;
            if (v < 0) v = 0;
            fb[m * nf + k] = v * enorm;
        }
    }
    free(all_freqs);
    free(f_pts);
}

void lfo_applysp(const lfo_cfgsp* c, const lfo_paramssp* p, const float* wav, int64_t L,
                 double* logmel, double* power) {
    const int n_fft = c->n_fft, nf = n_fft / 2 + 1, nm = c->n_mels, hop = c->hop;
    const int T = p->n_frames, pad = n_fft / 2, woff = (n_fft - c->win_length) / 2;
    double* win = (double*)calloc(n_fft, sizeof(double));
    for (int n = 0; n < c->win_length; n++)
        win[woff + n] = 0.5 - 0.5 * cos(2.0 * M_PI * n / c->win_length); /* periodic Hann */
    double* fb = (double*)malloc(sizeof(double) * nm * nf);
    lfo_mel_fbank(c, fb);
    double* cosv = (double*)malloc(sizeof(double) * n_fft);
    double* sinv = (double*)malloc(sizeof(double) * n_fft);
    for (int n = 0; n < n_fft; n++) {
        cosv[n] = cos(2.0 * M_PI * n / n_fft);
        sinv[n] = sin(2.0 * M_PI * n / n_fft);
    }
    double* frame = (double*)malloc(sizeof(double) * n_fft);
    double* pw = (double*)malloc(sizeof(double) * nf);
    for (int t = 0; t < T; t++) {
        for (int n = 0; n < n_fft; n++) {
            int64_t j = (int64_t)t * hop + n - pad; /* reflect pad */
            if (j < 0) j = -j;
            if (j >= L) j = 2 * (L - 1) - j;
            frame[n] = (double)wav[j] * win[n];
        }
        for (int k = 0; k < nf; k++) {
            double re = 0, im = 0;
            for (int n = 0; n < n_fft; n++) {
                int idx = (int)(((int64_t)k * n) % n_fft);
                re += frame[n] * cosv[idx];
                im -= frame[n] * sinv[idx];
            }
            pw[k] = re * re + im * im;
            if (power) power[(int64_t)k * T + t] = pw[k];
        }
        for (int m = 0; m < nm; m++) {
            double acc = 0;
            for (int k = 0; k < nf; k++) acc += fb[m * nf + k] * pw[k];
            logmel[(int64_t)m * T + t] = log(acc + c->log_eps);
        }
    }
    for (int i = 0; i < p->n_fmask; i++)
        for (int m = p->f_lo[i]; m < p->f_lo[i] + p->f_w[i]; m++)
            for (int t = 0; t < T; t++) logmel[(int64_t)m * T + t] = 0.0;
    for (int i = 0; i < p->n_tmask; i++)
        for (int t = p->t_lo[i]; t < p->t_lo[i] + p->t_w[i] && t < T; t++)
            for (int m = 0; m < nm; m++) logmel[(int64_t)m * T + t] = 0.0;
    free(win); free(fb); free(cosv); free(sinv); free(frame); free(pw);
}
