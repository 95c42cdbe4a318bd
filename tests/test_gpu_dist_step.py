"""The request-sharded decode step across processes: two ranks on the box's GPU(s)
(distinct GPUs when there are two: real NVLink peer mappings; else both on cuda:0, time-sliced),
CUDA-IPC peer-memory exchanges inside the goodput and update kernels, gloo for the handle
exchange.  Every rank's k*, goodput, alpha and outputs must equal the oracle's step on the union
of the requests (tests/dist_step_worker.py); then bench.py's N > 1 path (weak line + strong and
config-4 sub-objects) runs on the same two ranks and must print one well-formed JSON line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _torchrun(args, port, env=None, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port)] + args
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout, env=e)


def test_request_sharded_step_two_processes_equals_oracle():
    r = _torchrun([os.path.join(ROOT, "tests", "dist_step_worker.py")], 29541)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert r.stdout.count("DIST-STEP-OK") == 2, r.stdout[-4000:]


def test_bench_two_ranks_shared_gpu_json_line():
    import torch
    env = {} if torch.cuda.device_count() >= 2 else {"TSV_BENCH_SHARED_GPU": "1"}
    r = _torchrun(["bench.py", "--gpus", "2", "--steps", "64", "--warmup", "3", "--e2e-steps", "2", "--graph-steps", "16"],
                  29543, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-5000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0 and d["device_status"] == 0
    assert d["config"]["global_batch"] == 512 and "p2p" in d["config"]["parallelism"]
    s = d["workloads"]["strong"]
    assert "error" not in s, s
    assert s["scaling"] == "strong" and s["config"]["global_batch"] == 256 and s["value"] > 0 and s["device_status"] == 0
    c4 = d["workloads"]["config4"]
    assert c4["n_gpus"] == 2 and c4["config"]["vocab"] == 128256 and c4["value"] > 0 and c4["device_status"] == 0
    assert d["global_state_consistent"] is True
