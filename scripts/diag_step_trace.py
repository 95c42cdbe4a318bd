"""Diagnostic (not part of the product): timeline of the decode step's kernels on B200.

Builds libtsv with -DTSV_STEP_TRACE=1 (thread 0 of every CTA of lookup / choose-k / scan / race /
emit stamps %globaltimer at entry, after its grid-dependency wait and at exit), replays a CUDA graph
of 8 SpecStep steps (B = 256, V = 32000, L = 4096, both READY flags and the early trigger unless
--plain), and prints per step and kernel: first entry, first wait release, last exit (us from the
step's first lookup entry), and the critical path between consecutive kernels.
usage: python scripts/diag_step_trace.py [--plain]"""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
env = dict(os.environ, TSV_NVCC_EXTRA="-DTSV_STEP_TRACE=1")
subprocess.run([sys.executable, "-m", "paper_2406_14066_b200.build", "--force"], check=True, env=env, cwd=ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2406_14066_b200 import tsv  # noqa: E402
from paper_2406_14066_b200.step import SpecStep  # noqa: E402

plain = "--plain" in sys.argv
L = tsv.lib()
readers = [getattr(L, f"tsv_debug_step_trace_{n}") for n in ("lookup", "goodput", "verify")]
for r in readers:
    r.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
    r.restype = ctypes.c_uint32
buf = np.zeros((1 << 16, 6), np.uint64)


def read_all():
    ev = []
    for r in readers:
        n = r(buf.ctypes.data, 1 << 16)
        ev.append(buf[:n].copy())
    return np.concatenate(ev)


inp = synth.make_step_inputs(B=256, V=32000, L=4096, k_max=8, seed=240614066, device="cuda", sets=4)
st = SpecStep(inp, lookup_ready=not plain, early_trigger=not plain)
steps = list(range(8))
st.capture(steps)
for _ in range(3):
    st.replay()
torch.cuda.synchronize()
read_all()  # clear
st.replay()
torch.cuda.synchronize()
ev = read_all()
names = {0: "lookup", 1: "choose_k", 2: "scan", 3: "race", 4: "emit"}
per_launch = {0: 256, 1: 1, 2: 32, 3: None, 4: None}
ids = ev[:, 0] & 0xFF
t_in, t_wait, t_out = ev[:, 1].astype(np.int64), ev[:, 2].astype(np.int64), ev[:, 3].astype(np.int64)
launches = []
for k in range(5):
    sel = np.nonzero(ids == k)[0]
    sel = sel[np.argsort(t_in[sel])]
    n = per_launch[k] or len(sel) // len(steps)
    for j in range(len(steps)):
        s_ = sel[j * n:(j + 1) * n]
        w = t_wait[s_]
        m1, m2 = ev[s_, 4].astype(np.int64), ev[s_, 5].astype(np.int64)
        launches.append((j, k, t_in[s_].min(), w[w > 0].min() if (w > 0).any() else 0, t_out[s_].max(),
                         m1.max(), m2.max()))
launches.sort(key=lambda x: (x[0], x[1]))
t0 = min(l[2] for l in launches)
print(f"{'step':>4} {'kernel':>9} {'entry':>8} {'waited':>8} {'exit':>8} {'mark1':>8} {'mark2':>8}  (us from the first entry)")
for j, k, a, w, b, m1, m2 in launches:
    f = lambda x: (x - t0) / 1e3 if x else float("nan")  # noqa: E731
    print(f"{j:>4} {names[k]:>9} {f(a):8.2f} {f(w):8.2f} {f(b):8.2f} {f(m1):8.2f} {f(m2):8.2f}")
ends = [l[4] for l in launches if l[1] == 4]
print("emit-to-emit (us per step):", np.round(np.diff(ends) / 1e3, 2))
