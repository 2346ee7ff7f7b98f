"""N>1 plumbing of bench.py on CPU (gloo, world_size 2): the 2-D path runs
as independent replicas, so the only collectives are the
timing barrier and the max over ranks; the reference arm runs on rank 0 only.
"""
import json
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
from paper_2009_13840_b200.replicas import Replicas
r = Replicas("gloo")
r.barrier()
v = r.max_over_ranks(1.5 + r.rank)
print(json.dumps({"rank": r.rank, "ws": r.ws, "max": v}), flush=True)
r.close()
"""


def _torchrun(nproc, args, port, env_extra=None, timeout=300):
    env = dict(os.environ, ROOT=ROOT, **(env_extra or {}))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)


def test_replicas_max_over_ranks(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    r = _torchrun(2, [str(script)], 29631)
    assert r.returncode == 0, r.stderr[-2000:]
    # the two ranks share stdout: pick the JSON objects out of it
    lines = [json.loads(x) for x in re.findall(r"\{[^{}]*\}", r.stdout)]
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert all(x["ws"] == 2 and x["max"] == 2.5 for x in lines)


def test_replicas_single_process_is_identity():
    from paper_2009_13840_b200.replicas import Replicas

    r = Replicas("gloo")
    assert r.ws == 1 and r.max_over_ranks(3.25) == 3.25


def test_reference_arm_rank0_only():
    """bench.py --impl reference under torchrun N=2: one JSON line (rank 0),
    the other rank exits 0 without work."""
    r = _torchrun(2, ["bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                      "--warmup", "0", "--config", "config1"], 29633)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "reference"
