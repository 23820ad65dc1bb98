"""bench.py's multi-rank launcher on the CPU (no GPU needed): `--gpus 2` without
torchrun re-launches the script as two ranks (torch.distributed.run on 127.0.0.1, the
driver's launch form); the reference arm (the CPU oracle, this tier's reference) runs
on rank 0 behind a gloo group and prints one JSON line with n_gpus = 2."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra, env=None):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "gemv",
           "--steps", "1", "--warmup", "0", *extra]
    e = dict(os.environ, OMP_NUM_THREADS="2", **(env or {}))
    e.pop("WORLD_SIZE", None)
    e.pop("RANK", None)
    return subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=e, cwd=ROOT)


def test_bench_relaunches_two_ranks():
    r = _run("--gpus", "2")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1


def test_bench_single_rank_line():
    r = _run()
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["metric"].startswith("bitserial conv/GEMM binary TOPS")


def test_bench_world_mismatch_refused():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=120, cwd=ROOT,
                       env=dict(os.environ, WORLD_SIZE="3", RANK="0"))
    assert r.returncode != 0 and "WORLD_SIZE=3" in (r.stderr + r.stdout)
