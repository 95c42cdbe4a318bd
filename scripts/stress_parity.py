"""Randomised verify parity stress (diagnostic; the pinned cases are in tests/): random batch shapes,
vocab sizes, chunk widths, dense / one-hot q, prune on / off, every result against the oracle.
usage: python scripts/stress_parity.py [seconds] [--logits | --greedy] [--seed=N]
--logits: the fused softmax-from-logits verify (random temperatures) against the oracle's softmax rows +
verify; requests that differ are counted (near ties may flip, tests/test_gpu_parity.py lists them).
--greedy: the temperature-0 verify (drafts = the row argmax w.p. 0.7, ties from small-integer rows half the
time) against the oracle, bit-exact."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2406_14066_b200 import tsv  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
budget = float(args[0]) if args else 120.0
LOGITS = "--logits" in sys.argv
GREEDY = "--greedy" in sys.argv
seed_arg = [a for a in sys.argv if a.startswith("--seed=")]
rng = np.random.default_rng(int(seed_arg[0].split("=")[1]) if seed_arg else 12345)
t0, n, fails, req = time.time(), 0, 0, 0
while time.time() - t0 < budget:
    B = int(rng.integers(1, 200))
    V = int(rng.choice([int(rng.integers(1, 600)), int(rng.integers(600, 40000)), 32000, 4096 + int(rng.integers(0, 128))]))
    k_max = int(rng.integers(0, 9))
    dense = bool(rng.integers(0, 2))
    lam = float(rng.uniform(0.05, 0.98))
    chunk = int(rng.choice([0, 0, 128, 256, 384, 1024, 1792, 4096]))
    flags = tsv.VERIFY_NO_PRUNE if rng.random() < 0.15 else 0
    seed, step = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**32))
    if GREEDY:
        krng = np.random.default_rng(int(rng.integers(0, 2**31)))
        ks = krng.integers(0, k_max + 1, B)
        ro = np.zeros(B + 1, np.int32)
        ro[1:] = np.cumsum(ks + 1)
        ld = (V + 3) // 4 * 4
        if krng.random() < 0.5:
            p = krng.integers(0, 5, (int(ro[-1]), ld)).astype(np.float32)
        else:
            p = krng.standard_normal((int(ro[-1]), ld)).astype(np.float32)
        am = p[:, :V].argmax(axis=1)
        drafts = np.array([int(am[ro[i] + j]) if krng.random() < 0.7 else int(krng.integers(0, V))
                           for i in range(B) for j in range(ks[i])], np.int32)
        ona, oout, ost = oracle.verify_greedy(p, ro, drafts, k_max, vocab=V)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        dt = torch.tensor(drafts if len(drafts) else np.zeros(0, np.int32), dtype=torch.int32, device="cuda")
        na, out = tsv.tsv_verify_greedy(torch.tensor(p, device="cuda"), torch.tensor(ro, device="cuda"), dt, k_max,
                                        device_status=st, vocab=V, chunk=chunk)
        torch.cuda.synchronize()
        ok = (na.cpu().numpy() == ona).all() and (out.cpu().numpy() == oout).all() and int(st.item()) == ost
        n += 1
        req += B
        if not ok:
            fails += 1
            print(f"GREEDY MISMATCH B={B} V={V} k_max={k_max} chunk={chunk}")
        continue
    if LOGITS:
        tau = float(rng.choice([0.5, 0.8, 1.0, 1.3, 2.0]))
        vb = synth.make_logits_batch(B=B, V=V, k_max=k_max, lam=lam, seed=int(rng.integers(0, 2**31)), dense_q=dense)
        npf = (lambda t: None if t is None else t.detach().cpu().numpy())
        p = oracle.softmax_rows(npf(vb.p), tau, vocab=V)
        q = None if vb.q is None else oracle.softmax_rows(npf(vb.q), tau, vocab=V)
        ona, oout, ost = oracle.verify(p, q, npf(vb.row_offsets), npf(vb.draft_tokens),
                                       npf(vb.request_ids).view(np.uint32), seed, step, vb.k_max, vocab=V)
        g = vb.to("cuda")
        na, out = tsv.tsv_verify_accept_logits(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, seed, step,
                                               vb.k_max, temperature=tau, vocab=V)
        torch.cuda.synchronize()
        diff = int(((na.cpu().numpy() != ona) | (out.cpu().numpy() != oout).any(1)).sum())
        n += 1
        req += B
        fails += diff
        if diff:
            print(f"{diff} of {B} requests differ: V={V} k_max={k_max} dense={dense} lam={lam:.2f} tau={tau} seed={seed} step={step}")
        continue
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
    req += B
    n += 1
    if not ok:
        fails += 1
        print(f"MISMATCH B={B} V={V} k_max={k_max} dense={dense} lam={lam:.2f} chunk={chunk} flags={flags} seed={seed} step={step}")
what = "logits verify calls" if LOGITS else ("greedy verify calls" if GREEDY else "verify calls")
print(f"stress: {n} random {what} ({req} requests), {fails} {'differing requests' if LOGITS else 'mismatching calls'} "
      f"({time.time() - t0:.0f} s)")
sys.exit(1 if fails else 0)
