"""Diagnostic (TSV_COUNT_EXACT=1 build): exact race evaluations, prune candidates and quads raced per
verify call at config 2 (B = 256, V = 32000, lambda = 0.7).
usage: TSV_NVCC_EXTRA=-DTSV_COUNT_EXACT=1 python -m paper_2406_14066_b200.build --force; python scripts/diag_exact.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2406_14066_b200 import tsv  # noqa: E402

L = tsv.lib()
f = L.tsv_debug_exact_count
f.argtypes = [ctypes.c_void_p]
out = (ctypes.c_ulonglong * 4)()
for lam in (0.7, 0.3, 0.9):
    vb = synth.make_verify_batch(B=256, V=32000, k_max=8, lam=lam, seed=240614066, device="cuda")
    f(ctypes.cast(out, ctypes.c_void_p))
    for step in range(4):
        tsv.tsv_verify_accept(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 240614066, step, 8)
    torch.cuda.synchronize()
    f(ctypes.cast(out, ctypes.c_void_p))
    ex, cand, quads, went = out[0] / 4, out[1] / 4, out[2] / 4, out[3] / 4 / 32
    el = quads * 4  # the quad counter counts per lane
    print(f"lambda {lam}: per call exact evals {ex:.0f}, prune candidates {cand:.0f}, elements {el:.0f}; "
          f"candidates/element {cand / max(1, el):.4f}, exact/element {ex / max(1, el):.5f}, "
          f"exact per row (256 x ~1.6 rows) {ex / 418:.0f}; warp entries into the candidate path {went:.0f} "
          f"(of {quads / 32:.0f} warp-quads)")
