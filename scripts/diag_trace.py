"""Diagnostic (not part of the product): per-item timeline of verify_race_kernel on config 2.

Builds libtsv with -DTSV_TRACE=1 (globaltimer stamps per work item: after the meta load,
after streaming, after the end-of-item exchange), runs one verify after the L2 has been
flushed by three other input sets, and prints the timeline: when items start and end,
stream time by row type (residual p+q vs bonus p), and items in flight over time.
"""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
env = dict(os.environ, TSV_NVCC_EXTRA="-DTSV_TRACE=1 " + os.environ.get("TRACE_EXTRA", ""))
subprocess.run([sys.executable, "-m", "paper_2406_14066_b200.build", "--force"], check=True, env=env, cwd=ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2406_14066_b200 import tsv  # noqa: E402

L = tsv.lib()
L.tsv_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
L.tsv_debug_trace_clear.argtypes = []
dev = torch.device("cuda")
sets = [synth.make_verify_batch(B=256, V=32000, k_max=8, lam=0.7, seed=11 + s, device=dev) for s in range(4)]
chunk = int(os.environ.get("CHUNK", "0"))
outs = []
for vb in sets:
    na = torch.empty(256, dtype=torch.int32, device=dev)
    out = torch.empty((256, 9), dtype=torch.int32, device=dev)
    a = tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 5, 0, 8, na, out,
                             chunk=chunk)
    ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), dev)
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    outs.append((a, ws, na))
for rep in range(3):
    for a, _, _ in outs:
        tsv._check(L.tsv_verify_accept(ctypes.byref(a), None))
torch.cuda.synchronize()
res = []
for trial in range(3):
    tsv._check(L.tsv_debug_trace_clear())
    for a, _, _ in outs[1:]:  # flush L2 with the other sets
        tsv._check(L.tsv_verify_accept(ctypes.byref(a), None))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tsv._check(L.tsv_verify_accept(ctypes.byref(outs[0][0]), None))
    e1.record()
    torch.cuda.synchronize()
    buf = np.zeros((65536, 4), np.uint64)
    tsv._check(L.tsv_debug_trace(buf.ctypes.data, 65536))
    res.append((e0.elapsed_time(e1) * 1e3, buf))

for us, buf in res:
    used = buf[:, 2] > 0
    item_idx = np.nonzero(used)[0]
    t = buf[used].astype(np.int64)
    t0 = t[:, 0].min()
    start, sdone, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
    resid = (t[:, 3] & 1).astype(bool)
    print(f"verify call {us:.2f} us (events, incl. launch); items {used.sum()} "
          f"(residual {resid.sum()}, bonus {(~resid).sum()}); race span {end.max():.2f} us")
    for name, msk in (("residual", resid), ("bonus", ~resid)):
        d = sdone[msk] - start[msk]
        print(f"  {name:8s} start p50 {np.median(start[msk]):5.2f} p99 {np.percentile(start[msk], 99):5.2f} | "
              f"stream p10 {np.percentile(d, 10):5.2f} p50 {np.median(d):5.2f} p90 {np.percentile(d, 90):5.2f} | "
              f"finish p50 {np.median(end[msk] - sdone[msk]):5.2f} | end p50 {np.median(end[msk]):5.2f} "
              f"max {end[msk].max():5.2f} us")
    sm = ((t[:, 3] >> 1) & 0x7FFFFFFF).astype(np.int64)
    cta = (t[:, 3] >> 32).astype(np.int64)
    sm_max = np.array([end[sm == k].max() for k in np.unique(sm)])
    sm_spread = np.array([end[sm == k].max() - end[sm == k].min() for k in np.unique(sm)])
    cta_spread = np.array([end[cta == k].max() - end[cta == k].min() for k in np.unique(cta)])
    print(f"  per-SM last end: p10 {np.percentile(sm_max, 10):5.2f} p50 {np.median(sm_max):5.2f} "
          f"p90 {np.percentile(sm_max, 90):5.2f} max {sm_max.max():5.2f} | within-SM spread p50 "
          f"{np.median(sm_spread):5.2f} | within-CTA spread p50 {np.median(cta_spread):5.2f} us")
    slot = cta // int(os.environ.get("SLOT_CTAS", "148"))
    for sl in np.unique(slot):  # CTAs by launch slot (blockIdx // SMs)
        msk = slot == sl
        print(f"  CTA slot {sl}: items {msk.sum()} end p50 {np.median(end[msk]):5.2f} "
              f"p90 {np.percentile(end[msk], 90):5.2f} max {end[msk].max():5.2f} | stream p50 "
              f"{np.median((sdone - start)[msk]):5.2f}")
    wpc = int(os.environ.get("WARPS_PER_CTA", "16"))
    wic = item_idx % wpc  # first round: item = global warp id
    line = []
    for w in range(wpc):
        msk = wic == w
        line.append(f"{w}:{np.median(end[msk]):.1f}")
    print("  end p50 by warp-in-CTA:", " ".join(line))
    bins = np.arange(0, end.max() + 0.5, 0.5)
    inflight = [int(((start <= b) & (end > b)).sum()) for b in bins]
    print("  items in flight every 0.5 us:", inflight)
    # per-SM load vs finish: residual items (2x bytes) per SM against the SM's last item end
    sms = np.unique(sm)
    nres = np.array([resid[sm == k].sum() for k in sms])
    nit = np.array([(sm == k).sum() for k in sms])
    units = nit + nres  # bonus 1 unit, residual 2 units of bytes
    cc = np.corrcoef(units, sm_max)[0, 1]
    print(f"  per-SM byte units (items + residual items): min {units.min()} p50 {np.median(units):.0f} max {units.max()} "
          f"| corr(units, SM last end) {cc:.2f}; SM last end of the 10 lightest / heaviest SMs: "
          f"{np.mean(sm_max[np.argsort(units)[:10]]):.2f} / {np.mean(sm_max[np.argsort(units)[-10:]]):.2f} us; "
          f"per-SM mean end {np.mean([end[sm == k].mean() for k in sms]):.2f} us")
