"""The N > 1 bench flow (bench.py under torch.distributed.run, one rank per
GPU in the driver's runs) executed on ONE GPU: two ranks share cuda:0 and talk
over gloo (the SMAP_BENCH_ONE_GPU test hook; the numbers of such a run mean
nothing).  It checks the sharded flow end to end: every rank plans its omega_x
shard, the per-rank 56-byte records are all-gathered and combined on the
device, and the combined records equal the oracle's values for the whole
workloads (the bench line's checksum_ok and configs_sharded.*.checked_vs_oracle)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_on_one_gpu():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    env = dict(os.environ, SMAP_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29613", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--sustained-steps", "0"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]                  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"].endswith("x2")
    assert d["checksum_ok"] is True
    assert d["checksum"]["count"] == d["checksum"]["expected_count"]
    for name, e in d["configs_sharded"].items():
        assert e["checked_vs_oracle"] is True, name
        if name != "C4":                                        # two plans in flight, records combined per step
            assert e["two_plans"]["checked_vs_oracle"] is True, name
