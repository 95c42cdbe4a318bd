"""Randomised verify parity stress (diagnostic; the pinned cases are in tests/): random batch shapes,
vocab sizes, chunk widths, dense / one-hot q, prune on / off, with and without the fused alpha update,
every result against the oracle.  usage: python scripts/stress_parity.py [seconds]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2406_14066_b200 import tsv  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(12345)
t0, n, fails = time.time(), 0, 0
while time.time() - t0 < budget:
    B = int(rng.integers(1, 200))
    V = int(rng.choice([int(rng.integers(1, 600)), int(rng.integers(600, 40000)), 32000, 4096 + int(rng.integers(0, 128))]))
    k_max = int(rng.integers(0, 9))
    dense = bool(rng.integers(0, 2))
    lam = float(rng.uniform(0.05, 0.98))
    chunk = int(rng.choice([0, 0, 128, 256, 384, 1024, 1792, 4096]))
    flags = tsv.VERIFY_NO_PRUNE if rng.random() < 0.15 else 0
    seed, step = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**32))
    vb = synth.make_verify_batch(B=B, V=V, k_max=k_max, lam=lam, seed=int(rng.integers(0, 2**31)), dense_q=dense)
    g = vb.to("cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    na, out = tsv.tsv_verify_accept(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, seed, step, vb.k_max,
                                    device_status=st, vocab=vb.vocab, chunk=chunk, flags=flags)
    npf = (lambda t: None if t is None else t.detach().cpu().numpy())
    ona, oout, ost = oracle.verify(npf(vb.p), npf(vb.q), npf(vb.row_offsets), npf(vb.draft_tokens),
                                   npf(vb.request_ids).view(np.uint32), seed, step, vb.k_max, vocab=vb.vocab)
    torch.cuda.synchronize()
    ok = (na.cpu().numpy() == ona).all() and (out.cpu().numpy() == oout).all() and int(st.item()) == ost
    n += 1
    if not ok:
        fails += 1
        print(f"MISMATCH B={B} V={V} k_max={k_max} dense={dense} lam={lam:.2f} chunk={chunk} flags={flags} seed={seed} step={step}")
print(f"stress: {n} random verify calls, {fails} mismatches ({time.time() - t0:.0f} s)")
sys.exit(1 if fails else 0)
