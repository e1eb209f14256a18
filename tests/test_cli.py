"""`loadflow_b200 run | compare` -- the reference CLI's experiment commands
(proj/tools/loadflow_main.cpp:34-134) for the GPU loaders."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2509_10712_b200", "loadflow_b200")


@pytest.fixture(scope="module")
def cli():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_2509_10712_b200", "csrc")])
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_2509_10712_b200", "host")])
    return CLI


def test_cli_usage_and_config_errors(cli, tmp_path):
    r = subprocess.run([cli], capture_output=True, text=True)
    assert r.returncode == 1 and "usage" in r.stderr
    bad = tmp_path / "bad.ini"
    bad.write_text("[workload]\nname img_seg\n")
    r = subprocess.run([cli, "run", str(bad)], capture_output=True, text=True)
    assert r.returncode == 2 and "expected key = value" in r.stderr
    cfg = tmp_path / "c.ini"
    cfg.write_text("[pipeline]\nloader = pytorch\n")
    r = subprocess.run([cli, "run", str(cfg)], capture_output=True, text=True)
    assert r.returncode == 2 and "minato-gpu or sync-gpu" in r.stderr


@pytest.mark.gpu
def test_cli_run_and_compare_on_gpu(cli, tmp_path):
    """The reference img_seg stream (generate(spec): same ids and costs) through the GPU
    loaders: Minato exactly-once with slow samples classified, sync without; the Minato
    run completes no later and idles the trainer less; compare prints both."""
    cfg = os.path.join(ROOT, "configs", "img_seg_gpu.ini")
    reps = {}
    for loader in ("sync-gpu", "minato-gpu"):
        out = tmp_path / loader
        r = subprocess.run([cli, "run", cfg, "--loader", loader, "--out", str(out)],
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        assert "exactly_once=yes" in r.stdout
        reps[loader] = json.loads((out / "report.json").read_text())
        assert reps[loader]["samples"] == 400
    assert reps["sync-gpu"]["slow_rate"] == 0.0
    assert reps["minato-gpu"]["slow_rate"] > 0.0
    assert reps["minato-gpu"]["completion_ms"] <= reps["sync-gpu"]["completion_ms"] * 1.02
    r = subprocess.run([cli, "compare", str(tmp_path / "sync-gpu" / "report.json"),
                        str(tmp_path / "minato-gpu" / "report.json"), "--csv", str(tmp_path / "cmp.csv")],
                       capture_output=True, text=True)
    assert r.returncode == 0 and "minato-gpu" in r.stdout and (tmp_path / "cmp.csv").exists()


def test_cli_dropin_usage(cli):
    r = subprocess.run([cli, "dropin", "--bogus", "1"], capture_output=True, text=True)
    assert r.returncode == 2 and "unknown option" in r.stderr


@pytest.mark.gpu
def test_cli_dropin_coalesces_per_sample_submissions(cli):
    """The drop-in C++ path (run_minato_pipeline wiring, one process_sample per worker
    thread) delivers every sample exactly once; with coalescing its workers' samples
    share launch groups instead of one launch per sample."""
    res = {}
    for co in (0, 40):
        r = subprocess.run([cli, "dropin", "--samples", "4096", "--workers", "16", "--batch", "64",
                            "--group", "16", "--coalesce-us", str(co), "--max-seconds", "100"],
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        res[co] = json.loads(r.stdout.strip().splitlines()[-1])
        assert res[co]["exactly_once"] is True and res[co]["samples"] == 4096
    assert res[0]["samples_per_launch"] < 1.5
    assert res[40]["samples_per_launch"] > 2.0
    print(res)


@pytest.mark.gpu
def test_cli_speech_from_pcm_files(cli, tmp_path):
    """The reference speech stream from int16 PCM sample files (LFG_FILE_PCM16, the
    reference's 2-B samples, workloads.cpp:115) through reader threads, pinned slots,
    K0 and the speech kernel: exactly once, every sample delivered."""
    cfg = tmp_path / "speech_file.ini"
    text = open(os.path.join(ROOT, "configs", "speech_file.ini")).read()
    cfg.write_text(text.replace("[gpu]\n", f"[gpu]\ndata_dir = {tmp_path / 'data'}\n"))
    out = tmp_path / "speech"
    r = subprocess.run([cli, "run", str(cfg), "--out", str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "exactly_once=yes" in r.stdout
    rep = json.loads((out / "report.json").read_text())
    assert rep["samples"] == 4096
