"""GPU tests of the boundary's error contract and the step_counts output (include/tsv.h):
device-side data errors stay inside the caller's arrays and set TSV_DEVSTATUS_* bits, the
lookup reports bad contexts, step_counts = (sum m_i, sum tested_i) on every verify flavour, and
TSV_VERIFY_META_READY honours its contract inside a graph whose preceding kernels write the
batch.  Expected values come only from oracle/."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def tsv():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2406_14066_b200 import tsv as t
    return t


def _np(t):
    return t.detach().cpu().numpy()


def _counts(na, k):
    """(sum m, sum tested) over valid requests, tested = m + [m < k] (tsv.h step_counts, R18)."""
    v = na >= 0
    return int(na[v].sum()), int((na[v] + (na[v] < k[v])).sum())


def _oracle(vb, seed, step):
    return oracle.verify(_np(vb.p), None if vb.q is None else _np(vb.q), _np(vb.row_offsets), _np(vb.draft_tokens),
                         _np(vb.request_ids).view(np.uint32), seed, step, vb.k_max, vocab=vb.vocab)


# ------------------------------------------------------------------------------ step_counts
def test_step_counts_lazy_update_logits_greedy(tsv):
    vb = synth.make_verify_batch(B=96, V=8192, k_max=8, lam=0.6, seed=41)
    vb.draft_tokens[3] = 9000  # one bad request: excluded from the sums
    g = vb.to(DEV)
    k = _np(vb.k)
    ona, oout, _ = _oracle(vb, 7, 2)
    sc = torch.full((2,), -99, dtype=torch.int64, device=DEV)
    for _ in range(2):  # repeated calls: zeroed by every call
        na, out = tsv.tsv_verify_accept(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, 7, 2, 8, step_counts=sc)
        torch.cuda.synchronize()
        assert (_np(na) == ona).all() and tuple(_np(sc)) == _counts(ona, k)
    # fused verify + update (the update CTA beside the race; the counts from the emit kernel)
    na2 = torch.empty_like(na)
    out2 = torch.empty_like(out)
    sc.fill_(-5)
    a = tsv.make_verify_args(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, 7, 2, 8, na2, out2,
                             step_counts=sc, flags=tsv.VERIFY_META_READY)
    ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    alpha = torch.tensor([0.7], dtype=torch.float64, device=DEV)
    tsv.tsv_verify_accept_update(a, alpha, 0.9)
    torch.cuda.synchronize()
    assert tuple(_np(sc)) == _counts(ona, k)
    assert float(alpha.item()) == oracle.update(0.7, ona, _np(vb.row_offsets), decay=0.9)
    # greedy
    gna, _ = tsv.tsv_verify_greedy(g.p, g.row_offsets, g.draft_tokens, 8, step_counts=sc)
    torch.cuda.synchronize()
    wna, _, _ = oracle.verify_greedy(_np(vb.p), _np(vb.row_offsets), _np(vb.draft_tokens), 8)
    assert (_np(gna) == wna).all() and tuple(_np(sc)) == _counts(wna, k)
    # logits
    lb = synth.make_logits_batch(B=40, V=4096, k_max=6, lam=0.7, seed=42)
    gl = lb.to(DEV)
    lna, _ = tsv.tsv_verify_accept_logits(gl.p, gl.q, gl.row_offsets, gl.draft_tokens, gl.request_ids, 3, 1, 6,
                                          step_counts=sc)
    torch.cuda.synchronize()
    xna, _, _ = oracle.verify_logits(_np(lb.p), _np(lb.q), _np(lb.row_offsets), _np(lb.draft_tokens),
                                     _np(lb.request_ids).view(np.uint32), 3, 1, 6)
    assert (_np(lna) == xna).all() and tuple(_np(sc)) == _counts(xna, _np(lb.k))


def test_step_counts_sharded_flavours(tsv):
    vb = synth.make_verify_batch(B=30, V=4096, k_max=8, lam=0.7, seed=43)
    g = vb.to(DEV)
    ona, _, _ = _oracle(vb, 9, 4)
    want = _counts(ona, _np(vb.k))
    G, Vs = 2, 2048
    # dense partial -> (loopback gather) -> combine
    tuples = torch.zeros((G, int(g.p.shape[0]), tsv.SHARD_TUPLE_BYTES // 8), dtype=torch.int64, device=DEV)
    na = torch.empty(30, dtype=torch.int32, device=DEV)
    out = torch.empty((30, 9), dtype=torch.int32, device=DEV)
    sc = torch.full((2,), 77, dtype=torch.int64, device=DEV)
    for s in range(G):
        a = tsv.make_verify_args(g.p[:, s * Vs:(s + 1) * Vs], g.q[:, s * Vs:(s + 1) * Vs], g.row_offsets,
                                 g.draft_tokens, g.request_ids, 9, 4, 8, na, out, vocab=Vs, vocab_offset=s * Vs,
                                 vocab_global=4096, step_counts=sc)
        ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
        tsv.tsv_verify_shard_partial(a, tuples[s])
        torch.cuda.synchronize()
    a = tsv.make_verify_args(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, 9, 4, 8, na, out,
                             step_counts=sc)
    tsv.tsv_verify_shard_combine(a, tuples, G)
    torch.cuda.synchronize()
    assert (_np(na) == ona).all() and tuple(_np(sc)) == want
    # peer-memory lazy sharding, two loopback ranks: each rank's counts are the whole batch's
    lb = tsv.P2PLoopback(G, 32)
    try:
        scs, args = [], []
        for s in range(G):
            n_ = torch.empty(30, dtype=torch.int32, device=DEV)
            o_ = torch.empty((30, 9), dtype=torch.int32, device=DEV)
            c_ = torch.full((2,), -1, dtype=torch.int64, device=DEV)
            a = tsv.make_verify_args(g.p[:, s * Vs:(s + 1) * Vs], g.q[:, s * Vs:(s + 1) * Vs], g.row_offsets,
                                     g.draft_tokens, g.request_ids, 9, 4, 8, n_, o_, vocab=Vs, vocab_offset=s * Vs,
                                     vocab_global=4096, step_counts=c_)
            ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
            a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
            args.append((a, ws, n_, o_))  # keep every output buffer alive while the kernels write it
            scs.append(c_)
        for ph in range(3):
            for s in range(G):
                tsv.tsv_verify_shard_p2p_phase(args[s][0], lb.handles[s], ph)
        torch.cuda.synchronize()
        for s in range(G):
            assert (_np(args[s][2]) == ona).all() and tuple(_np(scs[s])) == want
    finally:
        lb.close()


# ------------------------------------------------------------------- offsets out of range
@pytest.mark.parametrize("offs,valid", [([0, 3, 6, 40], 2), ([0, 3, 9, 6], 1), ([0, 10, 3, 9], 0),
                                        ([0, 3, 6, 10], 2), ([0, 3, 3, 9], 1)])
@pytest.mark.parametrize("flavour", ["accept", "greedy", "logits"])
def test_offsets_out_of_range_are_flagged(tsv, offs, valid, flavour):
    # rows_p = 9 (B = 3, k = 2): an offset past rows_p, decreasing offsets, or rows reaching past the
    # 6 draft / q rows flag that request (-1, BAD_K) and the passes stay inside the arrays; the first
    # `valid` requests keep the oracle's outputs
    vb = synth.make_verify_batch(B=3, V=256, k_max=4, k_fixed=2, lam=0.7, seed=44)
    g = vb.to(DEV)
    ro = torch.tensor(offs, dtype=torch.int32, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    na = torch.full((3,), -7, dtype=torch.int32, device=DEV)
    out = torch.full((3, 5), -7, dtype=torch.int32, device=DEV)
    sub = synth.VerifyBatch(vb.p, vb.q, vb.row_offsets[:valid + 1], vb.draft_tokens, vb.request_ids[:valid],
                            vb.k[:valid], vb.vocab, 4)
    if flavour == "accept":
        tsv.tsv_verify_accept(g.p, g.q, ro, g.draft_tokens, g.request_ids, 1, 1, 4, na, out, st)
        wna, wout, _ = _oracle(sub, 1, 1) if valid else (np.zeros(0), np.zeros((0, 5)), 0)
    elif flavour == "greedy":
        tsv.tsv_verify_greedy(g.p, ro, g.draft_tokens, 4, na, out, st)
        wna, wout, _ = (oracle.verify_greedy(_np(vb.p), _np(vb.row_offsets)[:valid + 1], _np(vb.draft_tokens), 4)
                        if valid else (np.zeros(0), np.zeros((0, 5)), 0))
    else:
        lb = synth.make_logits_batch(B=3, V=256, k_max=4, lam=0.7, seed=44, k_list=[2, 2, 2])
        gl = lb.to(DEV)
        tsv.tsv_verify_accept_logits(gl.p, gl.q, ro, gl.draft_tokens, gl.request_ids, 1, 1, 4, num_accepted=na,
                                     out_tokens=out, device_status=st)
        wna, wout, _ = (oracle.verify_logits(_np(lb.p), _np(lb.q), _np(lb.row_offsets)[:valid + 1],
                                             _np(lb.draft_tokens), _np(lb.request_ids)[:valid].view(np.uint32), 1, 1, 4)
                        if valid else (np.zeros(0), np.zeros((0, 5)), 0))
    torch.cuda.synchronize()
    gna, gout = _np(na), _np(out)
    bad = offs != [0, 3, 6, 9]
    assert bool(int(st.item()) & tsv.DEVSTATUS_BAD_K) == bad
    assert (gna[valid:] == -1).all() and (gout[valid:] == -1).all()
    assert (gna[:valid] == wna).all() and (gout[:valid] == wout).all()


# ------------------------------------------------------------------------------ lookup
def test_lookup_bad_context_flagged(tsv):
    ctx = torch.tensor(np.arange(300) % 7, dtype=torch.int32, device=DEV)
    offs = torch.tensor([0, 100, 60, 300, 200], dtype=torch.int32, device=DEV)  # request 1 and 3 decreasing
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    pr, pl = tsv.tsv_propose_lookup(ctx, offs, 1, 3, 4, device_status=st)
    torch.cuda.synchronize()
    opr, opl = oracle.lookup(_np(ctx)[:100], np.array([0, 100], np.int32), 1, 3, 4)
    assert int(st.item()) == tsv.DEVSTATUS_BAD_CONTEXT
    assert _np(pl)[0] == opl[0] and (_np(pr)[0] == opr[0]).all()
    assert _np(pl)[1] == 0 and (_np(pr)[1] == -1).all() and _np(pl)[3] == 0
    # L > TSV_MAX_CONTEXT (2^20): the 20-bit end position would overflow -> no proposal, flagged
    L = (1 << 20) + 5
    big = torch.tensor(np.arange(L) % 11, dtype=torch.int32, device=DEV)
    st.zero_()
    pr, pl = tsv.tsv_propose_lookup(big, torch.tensor([0, L], dtype=torch.int32, device=DEV), 1, 4, 5,
                                    device_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == tsv.DEVSTATUS_BAD_CONTEXT and int(pl.item()) == 0
    # exactly TSV_MAX_CONTEXT is accepted and equals the oracle
    L = 1 << 20
    st.zero_()
    pr, pl = tsv.tsv_propose_lookup(big[:L], torch.tensor([0, L], dtype=torch.int32, device=DEV), 1, 4, 5,
                                    device_status=st)
    torch.cuda.synchronize()
    opr, opl = oracle.lookup(_np(big)[:L], np.array([0, L], np.int32), 1, 4, 5)
    assert int(st.item()) == 0 and (_np(pl) == opl).all() and (_np(pr) == opr).all()


# ----------------------------------------------------- META_READY under PDL inside a graph
def test_meta_ready_in_graph_after_pdl_writers(tsv):
    """tsv_sim_target's first kernel writes row_offsets and the drafts, its second (a PDL kernel)
    writes the p rows immediately before the verify; with TSV_VERIFY_META_READY the scan reads the
    offsets / drafts before its grid-dependency wait.  Captured in one graph and replayed with new
    proposals each time, the outputs must equal the oracle on what the graph wrote."""
    B, K, V = 48, 5, 4096
    rows_cap = B * (K + 1)
    rng = np.random.Generator(np.random.PCG64(45))
    proposals = torch.empty((B, K), dtype=torch.int32, device=DEV)
    k_req = torch.empty(B, dtype=torch.int32, device=DEV)
    alpha_true = torch.tensor([0.6], dtype=torch.float32, device=DEV)
    p = torch.empty((rows_cap, V), dtype=torch.float32, device=DEV)
    ro = torch.empty(B + 1, dtype=torch.int32, device=DEV)
    drafts = torch.empty(rows_cap, dtype=torch.int32, device=DEV)
    info = torch.empty(rows_cap, dtype=torch.int32, device=DEV)
    rids = torch.arange(B, dtype=torch.int32, device=DEV)
    na = torch.empty(B, dtype=torch.int32, device=DEV)
    out = torch.empty((B, K + 1), dtype=torch.int32, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    a = tsv.make_verify_args(p, None, ro, drafts, rids, 11, 3, K, na, out, st, flags=tsv.VERIFY_META_READY)
    a.rows_p = rows_cap
    ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    L = tsv.lib()

    def body(s):
        tsv._check(L.tsv_sim_target(proposals.data_ptr(), K, k_req.data_ptr(), B, alpha_true.data_ptr(), V, V,
                                    rows_cap, p.data_ptr(), ro.data_ptr(), drafts.data_ptr(), info.data_ptr(), s))
        tsv._check(L.tsv_verify_accept(tsv.ctypes.byref(a), s))

    side = torch.cuda.Stream()
    proposals.copy_(torch.tensor(rng.integers(0, V, (B, K)), dtype=torch.int32))
    k_req.copy_(torch.tensor(rng.integers(0, K + 1, B), dtype=torch.int32))
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        body(side.cuda_stream)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        body(side.cuda_stream)
    for rep in range(4):
        proposals.copy_(torch.tensor(rng.integers(0, V, (B, K)), dtype=torch.int32))
        k_req.copy_(torch.tensor(rng.integers(0, K + 1, B), dtype=torch.int32))
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        r = _np(ro)
        n = int(r[-1])
        ona, oout, ost = oracle.verify(_np(p)[:n], None, r, _np(drafts)[:n - B], _np(rids).view(np.uint32), 11, 3, K)
        assert (_np(na) == ona).all() and (_np(out) == oout).all(), rep
        assert int(st.item()) == 0
