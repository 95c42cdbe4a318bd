"""Worker of tests/test_gpu_sanitize.py: every concurrency-heavy path of libtsv at small sizes,
each checked against the oracle, meant to run under compute-sanitizer (memcheck, racecheck,
synccheck, initcheck).  Test infrastructure only (it imports oracle/).

Paths (VERDICT r01 "next round" item 2; SURVEY.md:257 test layer 4):
  step    config-1 step (lookup n=3 on 4 x 512, choose-k PLD, verify B=4 k=4 V=32000 with
          TSV_VERIFY_META_READY, the fused update CTA of the race kernel) eager and as a CUDA graph;
          config-3-shaped lookup (L=4096, n 1-4); the fused lookup + choose-k (last-CTA arrival
          counter, int64 atomics)
  p2p     peer-memory vocab sharding, G=2 loopback ranks over 3 epochs (LL words, epoch parity),
          and (one rank) the fused request-sharded choose-k / verify+update exchanges and the int64
          all-reduce (the sanitizer serialises kernels: no concurrent loopback ranks)
  shard   lazy (flags / race / emit) and dense (partial / combine) vocab sharding in loopback
  greedy  greedy verify (row-slot clear kernel + red.max argmax + emit)
  logits  fused softmax-from-logits verify (statistics pass, logits scan, LOGITS race)
  bad     device-side data errors: decreasing offsets, oversized row_offsets[B], bad tokens,
          decreasing lookup offsets (BAD_CONTEXT)

usage: python tests/sanitize_worker.py [path ...]     (default: all); prints SANITIZE-OK <path>."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2406_14066_b200 import tsv  # noqa: E402

DEV = torch.device("cuda", 0)


def _np(t):
    return t.detach().cpu().numpy()


def _oracle_verify(vb, seed, step):
    return oracle.verify(_np(vb.p), None if vb.q is None else _np(vb.q), _np(vb.row_offsets), _np(vb.draft_tokens),
                         _np(vb.request_ids).view(np.uint32), seed, step, vb.k_max, vocab=vb.vocab)


def path_step():
    from paper_2406_14066_b200.step import SpecStep, StepInputs
    # config 1: B = 4, k = 4, V = 32000, 512-token contexts, n = 3
    vb = synth.make_verify_batch(B=4, V=32000, k_max=4, k_fixed=4, lam=0.7, seed=1, device=DEV)
    c, o = synth.make_contexts(B=4, L=512, seed=1)
    inp = StepInputs([vb], [torch.tensor(c, device=DEV)], [torch.tensor(o, device=DEV)],
                     [torch.tensor(np.diff(o).astype(np.int32), device=DEV)], 4, n_min=3, n_max=3)
    st = SpecStep(inp, device=DEV)
    st.reset_state()
    st.run(step=5)
    torch.cuda.synchronize()
    opr, opl = oracle.lookup(c, o, 3, 3, 5)
    assert (_np(st.proposal_len) == opl).all() and (_np(st.proposals) == opr).all()
    ok, _ = oracle.choose_k(0.7, np.diff(o).astype(np.int32), opl, 5, oracle.POLICY_PLD, synth.SPEC_DESK_TARGET,
                            synth.SPEC_DESK_DRAFT, pld_cost_ms=0.05)
    assert int(st.k_star.item()) == ok
    ona, oout, _ = _oracle_verify(vb, synth.DEFAULT_SEED, 5)
    assert (_np(st.num_accepted) == ona).all() and (_np(st.out_tokens) == oout).all()
    want = oracle.update(0.7, ona, _np(vb.row_offsets), decay=0.9)
    assert float(st.alpha.item()) == want
    # the same step as a CUDA graph (PDL edges inside the graph; the fused lookup + choose-k with
    # TSV_LOOKUP_INPUTS_READY in a second step object)
    stf = SpecStep(inp, device=DEV, fused=True)
    stf.capture([6, 7])
    stf.reset_state()
    stf.replay()
    torch.cuda.synchronize()
    ona7, oout7, _ = _oracle_verify(vb, synth.DEFAULT_SEED, 7)
    assert (_np(stf.num_accepted) == ona7).all() and (_np(stf.out_tokens) == oout7).all()
    st.capture([6, 7])
    st.reset_state()
    st.replay()
    torch.cuda.synchronize()
    ona7, oout7, _ = _oracle_verify(vb, synth.DEFAULT_SEED, 7)
    assert (_np(st.num_accepted) == ona7).all() and (_np(st.out_tokens) == oout7).all()
    # config-3-shaped lookup (fewer requests: the sanitizer's slowdown), n 1-4
    c3, o3 = synth.make_contexts(B=24, L=4096, seed=3)
    pr, pl = tsv.tsv_propose_lookup(torch.tensor(c3, device=DEV), torch.tensor(o3, device=DEV), 1, 4, 5)
    opr3, opl3 = oracle.lookup(c3, o3, 1, 4, 5)
    assert (_np(pl) == opl3).all() and (_np(pr) == opr3).all()
    # fused lookup + choose-k (last-CTA arrival, exact int64 atomics)
    counter = tsv.lookup_choose_scratch(DEV)
    ctx_len = torch.tensor(np.diff(o3).astype(np.int32), device=DEV)
    alpha = torch.tensor([0.7], dtype=torch.float64, device=DEV)
    for rep in range(4):  # reps 2-3: TSV_LOOKUP_INPUTS_READY (everything before the grid-dependency wait)
        _, pl2, k2, _ = tsv.tsv_propose_lookup_choose_k(torch.tensor(c3, device=DEV), torch.tensor(o3, device=DEV),
                                                        1, 4, 5, alpha, ctx_len, synth.SPEC_DESK_TARGET, 0.05, counter,
                                                        flags=tsv.LOOKUP_INPUTS_READY if rep >= 2 else 0)
        torch.cuda.synchronize()
        ok3, _ = oracle.choose_k(0.7, np.diff(o3).astype(np.int32), opl3, 5, oracle.POLICY_PLD,
                                 synth.SPEC_DESK_TARGET, synth.SPEC_DESK_DRAFT, pld_cost_ms=0.05)
        assert int(k2.item()) == ok3 and (_np(pl2) == opl3).all()
        assert int(counter.abs().sum().item()) == 0


def path_p2p():
    vb = synth.make_verify_batch(B=12, V=4096, k_max=8, lam=0.7, seed=26)
    g = vb.to(DEV)
    G, Vs = 2, 2048
    lb = tsv.P2PLoopback(G, 16)
    try:
        for step in (3, 4, 5, 6, 7):  # both slot parities, advancing epochs; steps 6-7: keys pushed by the race
            fl = tsv.VERIFY_P2P_FUSED if step >= 6 else 0
            outs, args = [], []
            for s in range(G):
                lo = s * Vs
                na = torch.full((vb.B,), -7, dtype=torch.int32, device=DEV)
                out = torch.full((vb.B, vb.k_max + 1), -7, dtype=torch.int32, device=DEV)
                stt = torch.zeros(1, dtype=torch.int32, device=DEV)
                a = tsv.make_verify_args(g.p[:, lo:lo + Vs], g.q[:, lo:lo + Vs], g.row_offsets, g.draft_tokens,
                                         g.request_ids, 21, step, vb.k_max, na, out, device_status=stt, vocab=Vs,
                                         vocab_offset=lo, vocab_global=vb.vocab, flags=fl)
                ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
                a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
                args.append((a, ws))
                outs.append((na, out, stt))
            for phase in range(3):
                for s in range(G):
                    tsv.tsv_verify_shard_p2p_phase(args[s][0], lb.handles[s], phase)
            torch.cuda.synchronize()
            ona, oout, ost = _oracle_verify(vb, 21, step)
            for na, out, stt in outs:
                assert (_np(na) == ona).all() and (_np(out) == oout).all() and int(stt.item()) == ost
    finally:
        lb.close()
    # request-sharded global sums over peer memory, one rank (the sanitizer serialises kernels, so a
    # kernel that pushes and then polls cannot wait for a second loopback rank's kernel): the fused
    # choose-k, the standalone int64 all-reduce and the update CTA of the verify, 3 calls each
    comm = tsv.P2PComm(0, 1, B_max=16)
    try:
        ctx_len = torch.tensor(np.full(vb.B, 700, np.int32), device=DEV)
        cap = torch.tensor(np.arange(vb.B) % 6, dtype=torch.int32, device=DEV)
        stt = torch.zeros(1, dtype=torch.int32, device=DEV)
        for call in range(3):
            alpha = torch.tensor([0.3 + 0.2 * call], dtype=torch.float64, device=DEV)
            k, gp, _ = tsv.tsv_goodput_choose_k_sharded(alpha, ctx_len, cap, 5, tsv.POLICY_PLD, synth.SPEC_DESK_TARGET,
                                                        comm, synth.SPEC_DESK_DRAFT, 0.05, device_status=stt)
            data = torch.arange(12, dtype=torch.int64, device=DEV) * (call + 3) - 50
            want = _np(data)
            tsv.tsv_allreduce_i64_p2p(data, comm, device_status=stt)
            na = torch.empty(vb.B, dtype=torch.int32, device=DEV)
            out = torch.empty((vb.B, vb.k_max + 1), dtype=torch.int32, device=DEV)
            a = tsv.make_verify_args(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, 21, call, vb.k_max, na,
                                     out, device_status=stt)
            ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
            a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
            a2 = torch.tensor([0.7], dtype=torch.float64, device=DEV)
            tsv.tsv_verify_accept_update_p2p(a, a2, comm, 0.9)
            torch.cuda.synchronize()
            ok, og = oracle.choose_k(0.3 + 0.2 * call, _np(ctx_len), _np(cap), 5, oracle.POLICY_PLD,
                                     synth.SPEC_DESK_TARGET, synth.SPEC_DESK_DRAFT, pld_cost_ms=0.05)
            ona, oout, _ = _oracle_verify(vb, 21, call)
            assert int(k.item()) == ok and (_np(gp).view(np.uint64) == og.view(np.uint64)).all()
            assert (_np(data) == want).all() and int(stt.item()) == 0
            assert (_np(na) == ona).all() and (_np(out) == oout).all()
            assert float(a2.item()) == oracle.update(0.7, ona, _np(vb.row_offsets), decay=0.9)
    finally:
        comm.close()


def path_shard():
    vb = synth.make_verify_batch(B=10, V=4096, k_max=6, lam=0.7, seed=17)
    g = vb.to(DEV)
    G, Vs = 2, 2048
    ona, oout, _ = _oracle_verify(vb, 5, 2)
    # lazy: flags -> sum -> race -> max -> emit (loopback exchanges on the device)
    args, masks, keys, res = [], [], [], []
    for s in range(G):
        lo = s * Vs
        na = torch.empty(vb.B, dtype=torch.int32, device=DEV)
        out = torch.empty((vb.B, vb.k_max + 1), dtype=torch.int32, device=DEV)
        a = tsv.make_verify_args(g.p[:, lo:lo + Vs], g.q[:, lo:lo + Vs], g.row_offsets, g.draft_tokens,
                                 g.request_ids, 5, 2, vb.k_max, na, out, vocab=Vs, vocab_offset=lo,
                                 vocab_global=vb.vocab)
        ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
        args.append((a, ws))
        res.append((na, out))
        m = torch.empty(vb.B, dtype=torch.int64, device=DEV)
        tsv.tsv_verify_shard_flags(a, m)
        masks.append(m)
    msum = masks[0] + masks[1]
    for a, _ in args:
        k = torch.empty(2 * vb.B, dtype=torch.int64, device=DEV)
        tsv.tsv_verify_shard_race(a, msum, k)
        keys.append(k)
    u = torch.stack(keys).cpu().numpy().view(np.uint64)  # the exchange: element-wise u64 max
    kk = torch.tensor(np.maximum(u[0], u[1]).view(np.int64), device=DEV)
    for a, _ in args:
        tsv.tsv_verify_shard_emit(a, msum, kk)
    torch.cuda.synchronize()
    for na, out in res:
        assert (_np(na) == ona).all() and (_np(out) == oout).all()
    # dense: partial -> gather -> combine
    rows = int(args[0][0].rows_p)
    tuples = torch.zeros((G, rows, tsv.SHARD_TUPLE_BYTES // 8), dtype=torch.int64, device=DEV)
    for s, (a, _) in enumerate(args):
        tsv.tsv_verify_shard_partial(a, tuples[s])
    na, out = res[0]
    na.fill_(-7)
    a = tsv.make_verify_args(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, 5, 2, vb.k_max, na, out,
                             vocab=vb.vocab, vocab_global=vb.vocab)
    tsv.tsv_verify_shard_combine(a, tuples, G)
    torch.cuda.synchronize()
    assert (_np(na) == ona).all() and (_np(out) == oout).all()


def path_greedy():
    vb = synth.make_verify_batch(B=16, V=4099, k_max=8, lam=0.7, seed=3, dense_q=False)
    g = vb.to(DEV)
    am = g.p.argmax(1).to(torch.int32)
    ro = g.row_offsets.long()
    rows = torch.cat([torch.arange(int(ro[i]), int(ro[i + 1]) - 1) for i in range(vb.B)]).to(DEV)
    keep = torch.arange(rows.numel(), device=DEV) % 3 != 0
    d = torch.where(keep, am[rows], g.draft_tokens).contiguous()
    na, out = tsv.tsv_verify_greedy(g.p, g.row_offsets, d, vb.k_max)
    torch.cuda.synchronize()
    wna, wout, _ = oracle.verify_greedy(_np(g.p), _np(g.row_offsets), _np(d), vb.k_max)
    assert (_np(na) == wna).all() and (_np(out) == wout).all()


def path_logits():
    lb = synth.make_logits_batch(B=8, V=4096, k_max=6, lam=0.7, seed=2)
    g = lb.to(DEV)
    na, out = tsv.tsv_verify_accept_logits(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, 3, 1, lb.k_max)
    torch.cuda.synchronize()
    xna, xout, _ = oracle.verify_logits(_np(lb.p), _np(lb.q), _np(lb.row_offsets), _np(lb.draft_tokens),
                                        _np(lb.request_ids).view(np.uint32), 3, 1, lb.k_max)
    assert (_np(na) == xna).all() and (_np(out) == xout).all()


def path_bad():
    """Device-side data errors must stay inside the allocations (memcheck) and set status bits."""
    vb = synth.make_verify_batch(B=3, V=256, k_max=4, k_fixed=2, lam=0.7, seed=4)
    g = vb.to(DEV)
    rows_p = int(g.p.shape[0])  # 9
    for offs in ([0, 3, 9, 6], [0, 3, 6, 40], [0, 10, 3, 9]):  # decreasing / past rows_p / past the drafts
        ro = torch.tensor(offs, dtype=torch.int32, device=DEV)
        for fn in ("accept", "greedy", "logits"):
            st = torch.zeros(1, dtype=torch.int32, device=DEV)
            na = torch.empty(3, dtype=torch.int32, device=DEV)
            out = torch.empty((3, 5), dtype=torch.int32, device=DEV)
            if fn == "accept":
                tsv.tsv_verify_accept(g.p, g.q, ro, g.draft_tokens, g.request_ids, 1, 1, 4, na, out, st)
            elif fn == "greedy":
                tsv.tsv_verify_greedy(g.p, ro, g.draft_tokens, 4, na, out, st)
            else:
                tsv.tsv_verify_accept_logits(g.p, g.q, ro, g.draft_tokens, g.request_ids, 1, 1, 4,
                                             num_accepted=na, out_tokens=out, device_status=st)
            torch.cuda.synchronize()
            assert int(st.item()) & tsv.DEVSTATUS_BAD_K, (offs, fn)
    assert rows_p == 9
    # lookup: decreasing context offsets -> length 0 and the BAD_CONTEXT bit
    ctx = torch.arange(64, dtype=torch.int32, device=DEV) % 5
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    pr, pl = tsv.tsv_propose_lookup(ctx, torch.tensor([0, 40, 20, 64], dtype=torch.int32, device=DEV), 1, 3, 4,
                                    device_status=st)
    torch.cuda.synchronize()
    assert int(pl[1].item()) == 0 and int(st.item()) & tsv.DEVSTATUS_BAD_CONTEXT


PATHS = {"step": path_step, "p2p": path_p2p, "shard": path_shard, "greedy": path_greedy, "logits": path_logits,
         "bad": path_bad}


def main():
    torch.cuda.set_device(DEV)
    names = sys.argv[1:] or list(PATHS)
    for n in names:
        PATHS[n]()
        torch.cuda.synchronize()
        print(f"SANITIZE-OK {n}", flush=True)


if __name__ == "__main__":
    main()
