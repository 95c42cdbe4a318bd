"""GPU <-> oracle parity through the C ABI (libtsv.so via the ctypes binding).

Bit-exact on every integer output (accepted counts, emitted token ids, proposals,
proposal lengths, k*), bit-exact on the goodput values and the updated alpha
(same binary64 operation sequence on both sides).  Inputs come
from synth/ (seeded); expected values come only from oracle/.
"""
import os

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
    return None if t is None else t.detach().cpu().numpy()


def oracle_verify(vb, seed, step):
    return oracle.verify(_np(vb.p), _np(vb.q), _np(vb.row_offsets), _np(vb.draft_tokens),
                         _np(vb.request_ids).view(np.uint32), seed, step, vb.k_max, vocab=vb.vocab)


def gpu_verify(tsv, vb, seed, step, **kw):
    g = vb.to(DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    na, out = tsv.tsv_verify_accept(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, seed,
                                    step, vb.k_max, device_status=st, vocab=vb.vocab, **kw)
    torch.cuda.synchronize()
    return _np(na), _np(out), int(st.item())


def assert_verify_parity(tsv, vb, seed=240614066, step=0, **kw):
    ona, oout, ost = oracle_verify(vb, seed, step)
    gna, gout, gst = gpu_verify(tsv, vb, seed, step, **kw)
    bad = np.nonzero((ona != gna) | (oout != gout).any(1))[0]
    assert bad.size == 0, (f"{bad.size} requests differ, first {bad[:5]}: oracle m={ona[bad[:3]]} "
                           f"out={oout[bad[:3]]} gpu m={gna[bad[:3]]} out={gout[bad[:3]]}")
    assert gst == ost
    return ona, oout


# --------------------------------------------------------------------------- verify
def test_config1_dense(tsv):
    vb = synth.make_verify_batch(B=4, V=32000, k_max=4, k_fixed=4, lam=0.7, seed=1)
    for step in range(4):
        assert_verify_parity(tsv, vb, step=step)


def test_config2_full(tsv):
    vb = synth.make_verify_batch(B=256, V=32000, k_max=8, lam=0.7, seed=2)
    na, _ = assert_verify_parity(tsv, vb, step=0)
    assert (na >= 0).all()
    assert_verify_parity(tsv, vb, step=7)


@pytest.mark.parametrize("lam", [0.3, 0.9])
def test_config2_acceptance_levels(tsv, lam):
    vb = synth.make_verify_batch(B=128, V=32000, k_max=8, lam=lam, seed=3)
    assert_verify_parity(tsv, vb, step=1)


def test_one_hot_drafts(tsv):
    vb = synth.make_verify_batch(B=96, V=32000, k_max=5, lam=0.6, seed=4, dense_q=False)
    assert vb.q is None
    assert_verify_parity(tsv, vb, step=3)


@pytest.mark.parametrize("chunk", [128, 640, 1792, 4096, 16384])
def test_chunking_does_not_change_results(tsv, chunk):
    vb = synth.make_verify_batch(B=48, V=32000, k_max=8, lam=0.7, seed=5)
    assert_verify_parity(tsv, vb, step=2, chunk=chunk)


def test_prune_off_identical(tsv):
    vb = synth.make_verify_batch(B=64, V=32000, k_max=8, lam=0.7, seed=6)
    a = gpu_verify(tsv, vb, 11, 0)
    b = gpu_verify(tsv, vb, 11, 0, flags=tsv.VERIFY_NO_PRUNE)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    vb1 = synth.make_verify_batch(B=32, V=4099, k_max=3, lam=0.5, seed=7, dense_q=False)
    a = gpu_verify(tsv, vb1, 11, 5)
    b = gpu_verify(tsv, vb1, 11, 5, flags=tsv.VERIFY_NO_PRUNE)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()


@pytest.mark.parametrize("V", [1, 3, 7, 13, 4096 + 3])
def test_ragged_vocab_sizes(tsv, V):
    vb = synth.make_verify_batch(B=16, V=V, k_max=6, lam=0.7, seed=8 + V)
    assert_verify_parity(tsv, vb, step=V)
    vb = synth.make_verify_batch(B=16, V=V, k_max=6, lam=0.7, seed=9 + V, dense_q=False)
    assert_verify_parity(tsv, vb, step=V)


def test_padded_ld(tsv):
    vb = synth.make_verify_batch(B=20, V=1000, k_max=4, lam=0.7, seed=10, ld=1032)
    vb.p[:, 1000:] = 5.0  # never read
    vb.q[:, 1000:] = 5.0
    assert_verify_parity(tsv, vb, step=1)


def test_k_zero_and_k_max(tsv):
    ks = [0] * 8 + [15] * 8
    vb = synth.make_verify_batch(B=16, V=2048, k_max=15, lam=0.95, seed=12, k_list=ks)
    assert_verify_parity(tsv, vb, step=0)


def _adversarial_batch():
    """Hand-built rows: p == q, zero rows, denormals, q(x)=0, p(x)=0, drafts at 0 and V-1."""
    V = 260
    rng = np.random.Generator(np.random.PCG64(13))
    rows_p, rows_q, drafts, ks = [], [], [], []

    def soft():
        z = rng.standard_normal(V) * 3
        e = np.exp(z - z.max())
        return (e / e.sum()).astype(np.float32)

    cases = []
    # 1. p == q (accept always; residual zero only by rounding)
    p = soft(); cases.append(([p, p, soft()], [p, p], [0, V - 1]))
    # 2. residual identically zero -> fallback (q >= p everywhere, unnormalised)
    p = soft(); q = p * 2; cases.append(([p, soft()], [q], [5]))
    # 3. denormal weights
    p = np.full(V, 1e-40, np.float32); p[3] = 2e-40; cases.append(([p], [], []))
    # 4. q(x) = 0 -> always accept
    p = soft(); q = soft(); q[7] = 0; cases.append(([p, soft()], [q], [7]))
    # 5. p(x) = 0 -> always reject
    p = soft(); p[9] = 0; q = soft(); cases.append(([p, soft()], [q], [9]))
    # 6. exact ties: all-equal weights
    p = np.full(V, 1.0 / V, np.float32); cases.append(([p], [], []))
    # 7. zero bonus row -> NO_WEIGHT
    cases.append(([np.zeros(V, np.float32)], [], []))
    # 8. single nonzero entry at V-1 and at 0
    p = np.zeros(V, np.float32); p[V - 1] = 1; cases.append(([p], [], []))
    p = np.zeros(V, np.float32); p[0] = 1; cases.append(([p], [], []))
    # 9. NaN in the residual row (NaN weight -> 0)
    p = soft(); q = soft(); p[11] = np.nan; cases.append(([p, soft()], [q], [12]))
    for pr, qr, d in cases:
        rows_p += pr; rows_q += qr; drafts += d; ks.append(len(d))
    B = len(ks)
    ro = np.zeros(B + 1, np.int32); ro[1:] = np.cumsum(np.array(ks) + 1)
    return synth.VerifyBatch(torch.tensor(np.stack(rows_p)), torch.tensor(np.stack(rows_q)),
                             torch.tensor(ro), torch.tensor(np.array(drafts, np.int32)),
                             torch.arange(B, dtype=torch.int32), torch.tensor(ks, dtype=torch.int32),
                             V, 2)


def test_adversarial_rows(tsv):
    vb = _adversarial_batch()
    for step in range(6):
        assert_verify_parity(tsv, vb, step=step)
        assert_verify_parity(tsv, vb, step=step, chunk=1024)


def test_bad_token_and_bad_k_flagged(tsv):
    vb = synth.make_verify_batch(B=8, V=512, k_max=3, lam=0.7, seed=14, k_fixed=3)
    vb.draft_tokens[4] = 512          # out of range (request 1)
    _, out, st = gpu_verify(tsv, vb, 1, 0)
    ona, oout, ost = oracle_verify(vb, 1, 0)
    assert (out == oout).all() and st & tsv.DEVSTATUS_BAD_TOKEN and ost & oracle.STATUS_BAD_TOKEN
    vb2 = synth.make_verify_batch(B=8, V=512, k_max=5, lam=0.7, seed=14, k_fixed=5)
    vb2.k_max = 3                      # every request has k = 5 > k_max
    _, out, st = gpu_verify(tsv, vb2, 1, 0)
    assert (out == -1).all() and st & tsv.DEVSTATUS_BAD_K


def test_repeated_calls_deterministic(tsv):
    vb = synth.make_verify_batch(B=64, V=32000, k_max=8, lam=0.7, seed=15).to(DEV)
    na = torch.empty(64, dtype=torch.int32, device=DEV)
    out = torch.empty((64, 9), dtype=torch.int32, device=DEV)
    a = tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 3, 4, 8, na, out)
    ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
    res = []
    for _ in range(3):
        tsv.tsv_verify_accept(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 3, 4, 8,
                              num_accepted=na, out_tokens=out, workspace=ws)
        torch.cuda.synchronize()
        res.append(out.clone())
    assert all((r == res[0]).all() for r in res)


def test_request_order_invariance(tsv):
    # outputs depend on request ids, not batch positions
    vb = synth.make_verify_batch(B=32, V=4096, k_max=4, lam=0.7, seed=16, k_fixed=4)
    na, out, _ = gpu_verify(tsv, vb, 5, 1)
    perm = torch.randperm(32, generator=torch.Generator().manual_seed(0))
    rows = vb.p.view(32, 5, -1)[perm].reshape(160, -1)
    qrows = vb.q.view(32, 4, -1)[perm].reshape(128, -1)
    d = vb.draft_tokens.view(32, 4)[perm].reshape(-1)
    vbp = synth.VerifyBatch(rows.contiguous(), qrows.contiguous(), vb.row_offsets, d.contiguous(),
                            vb.request_ids[perm].contiguous(), vb.k, vb.vocab, vb.k_max)
    na2, out2, _ = gpu_verify(tsv, vbp, 5, 1)
    assert (out2 == out[perm.numpy()]).all()


# ------------------------------------------------------------------ vocab-shard loopback
def shard_loopback(tsv, vb, G, seed, step, chunk=0):
    g = vb.to(DEV)
    B, V = vb.B, vb.vocab
    assert V % (4 * G) == 0
    Vs = V // G
    rows = g.p.shape[0]
    tuples = torch.zeros((G, rows, tsv.SHARD_TUPLE_BYTES // 8), dtype=torch.int64, device=DEV)
    na = torch.empty(B, dtype=torch.int32, device=DEV)
    out = torch.empty((B, vb.k_max + 1), dtype=torch.int32, device=DEV)
    for s in range(G):
        lo = s * Vs
        a = tsv.make_verify_args(g.p[:, lo:lo + Vs], None if g.q is None else g.q[:, lo:lo + Vs],
                                 g.row_offsets, g.draft_tokens, g.request_ids, seed, step, vb.k_max,
                                 na, out, vocab=Vs, vocab_offset=lo, vocab_global=V, chunk=chunk)
        ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
        a.workspace = ws.data_ptr()
        a.workspace_bytes = ws.numel()
        tsv.tsv_verify_shard_partial(a, tuples[s])
        torch.cuda.synchronize()
    a = tsv.make_verify_args(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, seed, step,
                             vb.k_max, na, out, vocab=V, vocab_global=V)
    tsv.tsv_verify_shard_combine(a, tuples, G)
    torch.cuda.synchronize()
    return _np(na), _np(out)


def _u64max(a, b):
    """Element-wise unsigned max of int64 tensors holding u64 bit patterns."""
    flip = torch.tensor(-(2 ** 63), dtype=torch.int64, device=a.device)
    return torch.maximum(a ^ flip, b ^ flip) ^ flip


def lazy_shard_loopback(tsv, vb, G, seed, step, chunk=0):
    """Two-round lazy sharding on one device: flags (sum) -> race (max) -> emit."""
    g = vb.to(DEV)
    B, V = vb.B, vb.vocab
    assert V % (4 * G) == 0
    Vs = V // G
    na = torch.empty(B, dtype=torch.int32, device=DEV)
    out = torch.empty((B, vb.k_max + 1), dtype=torch.int32, device=DEV)
    args = []
    for s in range(G):
        lo = s * Vs
        a = tsv.make_verify_args(g.p[:, lo:lo + Vs], None if g.q is None else g.q[:, lo:lo + Vs],
                                 g.row_offsets, g.draft_tokens, g.request_ids, seed, step, vb.k_max,
                                 na, out, vocab=Vs, vocab_offset=lo, vocab_global=V, chunk=chunk)
        ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
        a.workspace = ws.data_ptr()
        a.workspace_bytes = ws.numel()
        args.append((a, ws))
    masks = torch.zeros(B, dtype=torch.int64, device=DEV)
    for a, _ in args:
        m = torch.empty(B, dtype=torch.int64, device=DEV)
        tsv.tsv_verify_shard_flags(a, m)
        masks += m
    keys = torch.zeros(2 * B, dtype=torch.int64, device=DEV)
    for a, _ in args:
        k = torch.empty(2 * B, dtype=torch.int64, device=DEV)
        tsv.tsv_verify_shard_race(a, masks, k)
        keys = _u64max(keys, k)
    tsv.tsv_verify_shard_emit(args[0][0], masks, keys)
    torch.cuda.synchronize()
    return _np(na), _np(out)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_lazy_vocab_shard_loopback_equals_oracle(tsv, G):
    vb = synth.make_verify_batch(B=64, V=32000, k_max=8, lam=0.7, seed=24)
    ona, oout, _ = oracle_verify(vb, 21, 3)
    na, out = lazy_shard_loopback(tsv, vb, G, 21, 3)
    assert (na == ona).all() and (out == oout).all()


def test_lazy_vocab_shard_one_hot_and_adversarial(tsv):
    vb = synth.make_verify_batch(B=40, V=4096, k_max=6, lam=0.7, seed=25, dense_q=False)
    ona, oout, _ = oracle_verify(vb, 2, 2)
    for G in (2, 4):
        na, out = lazy_shard_loopback(tsv, vb, G, 2, 2, chunk=1024)
        assert (na == ona).all() and (out == oout).all()
    adv = _adversarial_batch()
    adv.vocab = 256
    adv.p = adv.p[:, :256].contiguous(); adv.q = adv.q[:, :256].contiguous()
    adv.draft_tokens = adv.draft_tokens.clamp(max=255)
    for step in range(4):
        ona, oout, _ = oracle_verify(adv, 4, step)
        na, out = lazy_shard_loopback(tsv, adv, 4, 4, step)
        assert (na == ona).all() and (out == oout).all()


def p2p_shard_loopback(tsv, vb, G, seed, steps, chunk=0, B_max=None, flags=0, bounds=None):
    """Lazy two rounds over peer memory (tsv_verify_shard_p2p_phase), G virtual ranks on one device:
    all ranks phase 0, then phase 1, then phase 2, for each step; every rank's outputs are returned.
    flags: e.g. VERIFY_P2P_FUSED (the race items push their chunk keys; no keys kernel).
    bounds: explicit shard column boundaries [0, ..., V] (default: G equal shards)."""
    g = vb.to(DEV)
    B, V = vb.B, vb.vocab
    if bounds is None:
        assert V % (4 * G) == 0
        bounds = [s * (V // G) for s in range(G)] + [V]
    lb = tsv.P2PLoopback(G, B_max or max(B, 1))
    res = []
    try:
        for step in steps:
            outs, args = [], []
            for s in range(G):
                lo, Vs = bounds[s], bounds[s + 1] - bounds[s]
                na = torch.full((B,), -7, dtype=torch.int32, device=DEV)
                out = torch.full((B, vb.k_max + 1), -7, dtype=torch.int32, device=DEV)
                st = torch.zeros(1, dtype=torch.int32, device=DEV)
                a = tsv.make_verify_args(g.p[:, lo:lo + Vs], None if g.q is None else g.q[:, lo:lo + Vs],
                                         g.row_offsets, g.draft_tokens, g.request_ids, seed, step, vb.k_max,
                                         na, out, device_status=st, vocab=Vs, vocab_offset=lo, vocab_global=V,
                                         chunk=chunk, flags=flags)
                ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
                a.workspace = ws.data_ptr()
                a.workspace_bytes = ws.numel()
                args.append((a, ws))
                outs.append((na, out, st))
            for phase in range(3):
                for s in range(G):
                    tsv.tsv_verify_shard_p2p_phase(args[s][0], lb.handles[s], phase)
            torch.cuda.synchronize()
            res.append([(_np(na), _np(out), int(st.item())) for na, out, st in outs])
    finally:
        lb.close()
    return res


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_p2p_vocab_shard_loopback_equals_oracle(tsv, G, fused):
    # three consecutive calls: both slot parities and advancing epochs
    vb = synth.make_verify_batch(B=64, V=32000, k_max=8, lam=0.7, seed=26)
    res = p2p_shard_loopback(tsv, vb, G, 21, [3, 4, 5], B_max=80, flags=tsv.VERIFY_P2P_FUSED if fused else 0)
    for step, ranks in zip([3, 4, 5], res):
        ona, oout, ost = oracle_verify(vb, 21, step)
        for na, out, st in ranks:
            assert (na == ona).all() and (out == oout).all() and st == ost


@pytest.mark.parametrize("fused", [False, True])
def test_p2p_vocab_shard_one_hot_adversarial_llama3(tsv, fused):
    fl = tsv.VERIFY_P2P_FUSED if fused else 0
    vb = synth.make_verify_batch(B=40, V=4096, k_max=6, lam=0.7, seed=27, dense_q=False)
    ona, oout, _ = oracle_verify(vb, 2, 2)
    for G in (2, 4):
        for na, out, st in p2p_shard_loopback(tsv, vb, G, 2, [2], chunk=1024, flags=fl)[0]:
            assert (na == ona).all() and (out == oout).all()
    adv = _adversarial_batch()  # includes p == q rows: a residual zero on every rank (R5 fallback path)
    adv.vocab = 256
    adv.p = adv.p[:, :256].contiguous(); adv.q = adv.q[:, :256].contiguous()
    adv.draft_tokens = adv.draft_tokens.clamp(max=255)
    res = p2p_shard_loopback(tsv, adv, 4, 4, [0, 1, 2, 3], flags=fl)
    for step, ranks in enumerate(res):
        ona, oout, ost = oracle_verify(adv, 4, step)
        for na, out, st in ranks:
            assert (na == ona).all() and (out == oout).all() and st == ost
    vb3 = synth.make_verify_batch(B=24, V=128256, k_max=8, lam=0.7, seed=28)  # Llama-3 vocabulary, G = 8
    ona, oout, _ = oracle_verify(vb3, 9, 1)
    for na, out, st in p2p_shard_loopback(tsv, vb3, 8, 9, [1], flags=fl)[0]:
        assert (na == ona).all() and (out == oout).all()


@pytest.mark.slow
def test_config4_full_size_unsharded_and_p2p_g8(tsv):
    # BASELINE config 4 at its full size (B = 256, k in 0..8, V = 128256): the unsharded call (with
    # TSV_VERIFY_META_READY, as the bench times it) and eight loopback vocab shards over peer memory,
    # LL keys kernel and fused push, every request equal to the oracle
    vb = synth.make_verify_batch(B=256, V=128256, k_max=8, lam=0.7, seed=240614066)
    ona, oout = assert_verify_parity(tsv, vb, 240614066, 0, flags=tsv.VERIFY_META_READY)
    for fl in (0, tsv.VERIFY_P2P_FUSED):
        for na, out, st in p2p_shard_loopback(tsv, vb, 8, 240614066, [0], flags=fl)[0]:
            assert (na == ona).all() and (out == oout).all() and st == 0


def test_p2p_fused_uneven_shards(tsv):
    # fused push with shards of 2052 and 2048 columns (V = 4100), chunk 512: every rank polls
    # NC = 5 chunk slots per rank; rank 1 races only 4 chunks and its flags kernel fills the fifth slot
    vb = synth.make_verify_batch(B=30, V=4100, k_max=8, lam=0.6, seed=33)
    res = p2p_shard_loopback(tsv, vb, 2, 5, [0, 1, 2], chunk=512, flags=tsv.VERIFY_P2P_FUSED, bounds=[0, 2052, 4100])
    for step, ranks in enumerate(res):
        ona, oout, ost = oracle_verify(vb, 5, step)
        for na, out, st in ranks:
            assert (na == ona).all() and (out == oout).all() and st == ost
    # a shard needing more chunks than NC = ceil(ceil4(vocab_global / world) / chunk) is refused on the host
    with pytest.raises(RuntimeError):
        p2p_shard_loopback(tsv, vb, 2, 5, [0], chunk=512, flags=tsv.VERIFY_P2P_FUSED, bounds=[0, 2600, 4100])


@pytest.mark.parametrize("fused", [False, True])
def test_p2p_graph_replay_advances_epochs(tsv, fused):
    # the call epoch lives on the device: a captured graph of 3 calls replayed twice stays correct
    vb = synth.make_verify_batch(B=32, V=8192, k_max=8, lam=0.7, seed=30)
    g = vb.to(DEV)
    comm = tsv.P2PComm(0, 1, B_max=32)
    try:
        outs = []
        args = []
        for step in range(3):
            na = torch.empty(vb.B, dtype=torch.int32, device=DEV)
            out = torch.full((vb.B, vb.k_max + 1), -7, dtype=torch.int32, device=DEV)
            a = tsv.make_verify_args(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, 8, step, vb.k_max,
                                     na, out, vocab=vb.vocab, vocab_global=vb.vocab,
                                     flags=tsv.VERIFY_P2P_FUSED if fused else 0)
            ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
            a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
            args.append((a, ws))
            outs.append((na, out))
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            tsv.tsv_verify_accept_sharded_p2p(args[0][0], comm, stream=side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            for a, _ in args:
                tsv.tsv_verify_accept_sharded_p2p(a, comm, stream=side)
        for _ in range(2):
            for na, out in outs:
                out.fill_(-7)
            graph.replay()
            torch.cuda.synchronize()
            for step, (na, out) in enumerate(outs):
                ona, oout, _ = oracle_verify(vb, 8, step)
                assert (_np(na) == ona).all() and (_np(out) == oout).all()
    finally:
        comm.close()


def test_p2p_vocab_shard_two_processes_ipc(tmp_path):
    # the real multi-process path (CUDA IPC buffers, system-scope flags, epochs) with two ranks on the one
    # GPU of this box (time-sliced contexts), over gloo for the handle exchange; each rank checks the oracle
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "tests", "p2p_worker.py")]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("P2P-OK") == 2, r.stdout[-3000:]


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_vocab_shard_loopback_equals_oracle(tsv, G):
    vb = synth.make_verify_batch(B=64, V=32000, k_max=8, lam=0.7, seed=17)
    ona, oout, _ = oracle_verify(vb, 21, 3)
    na, out = shard_loopback(tsv, vb, G, 21, 3)
    assert (na == ona).all() and (out == oout).all()


def test_vocab_shard_loopback_one_hot_and_adversarial(tsv):
    vb = synth.make_verify_batch(B=40, V=4096, k_max=6, lam=0.7, seed=18, dense_q=False)
    ona, oout, _ = oracle_verify(vb, 2, 2)
    for G in (2, 4):
        na, out = shard_loopback(tsv, vb, G, 2, 2, chunk=1024)
        assert (na == ona).all() and (out == oout).all()
    adv = _adversarial_batch()
    adv.vocab = 256
    adv.p = adv.p[:, :256].contiguous(); adv.q = adv.q[:, :256].contiguous()
    adv.draft_tokens = adv.draft_tokens.clamp(max=255)
    ona, oout, _ = oracle_verify(adv, 4, 1)
    na, out = shard_loopback(tsv, adv, 4, 4, 1)
    assert (na == ona).all() and (out == oout).all()


def test_verify_accept_sharded_nccl_world1(tsv):
    # partial -> ncclAllGather of the shard tuples -> combine, on a one-rank communicator
    vb = synth.make_verify_batch(B=64, V=32000, k_max=8, lam=0.7, seed=23)
    ona, oout, _ = oracle_verify(vb, 5, 9)
    g = vb.to(DEV)
    na = torch.empty(vb.B, dtype=torch.int32, device=DEV)
    out = torch.empty((vb.B, vb.k_max + 1), dtype=torch.int32, device=DEV)
    a = tsv.make_verify_args(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, 5, 9, vb.k_max, na, out,
                             vocab=vb.vocab, vocab_global=vb.vocab)
    comm = tsv.Comm(0, 1)
    try:
        ws = tsv.alloc_workspace(tsv.tsv_verify_sharded_workspace_size(a, 1), DEV)
        a.workspace = ws.data_ptr()
        a.workspace_bytes = ws.numel()
        for flags in (0, tsv.VERIFY_SHARD_DENSE):  # lazy two rounds (default), one-round dense
            na.fill_(-7)
            out.fill_(-7)
            a.flags = flags
            tsv.tsv_verify_accept_sharded(a, comm)
            torch.cuda.synchronize()
            assert (_np(na) == ona).all() and (_np(out) == oout).all(), flags
    finally:
        comm.close()


@pytest.mark.slow
def test_config4_llama3_vocab_sharded(tsv):
    # V = 128256 (Llama-3), B = 256, ragged k: one-round dense shard partials, G = 2/4/8
    vb = synth.make_verify_batch(B=256, V=128256, k_max=8, lam=0.7, seed=19)
    ona, oout, _ = oracle_verify(vb, 240614066, 0)
    gna, gout, _ = gpu_verify(tsv, vb, 240614066, 0)
    assert (gna == ona).all() and (gout == oout).all()
    for G in (2, 4, 8):
        na, out = shard_loopback(tsv, vb, G, 240614066, 0)
        assert (na == ona).all() and (out == oout).all()
        na, out = lazy_shard_loopback(tsv, vb, G, 240614066, 0)
        assert (na == ona).all() and (out == oout).all()


# --------------------------------------------------------------------------- lookup
def gpu_lookup(tsv, ctx, offs, n_min, n_max, K):
    c = torch.tensor(ctx, device=DEV)
    o = torch.tensor(offs, device=DEV)
    pr, pl = tsv.tsv_propose_lookup(c, o, n_min, n_max, K)
    torch.cuda.synchronize()
    return _np(pr), _np(pl)


def assert_lookup_parity(tsv, ctx, offs, n_min, n_max, K):
    opr, opl = oracle.lookup(ctx, offs, n_min, n_max, K)
    gpr, gpl = gpu_lookup(tsv, ctx, offs, n_min, n_max, K)
    assert (opl == gpl).all(), np.nonzero(opl != gpl)[0][:5]
    assert (opr == gpr).all()
    return opl


def test_lookup_inputs_ready_flag_in_pdl_chain(tsv):
    # TSV_LOOKUP_INPUTS_READY: the search runs before the grid-dependency wait.  Inside a captured graph,
    # right after a verify call (three PDL kernels) and followed by choose-k, the proposals must equal
    # the oracle's, on ragged contexts (short, empty, misaligned starts) and on config-3 contexts.
    vb = synth.make_verify_batch(B=64, V=32000, k_max=8, lam=0.7, seed=5).to(DEV)
    na = torch.empty(64, dtype=torch.int32, device=DEV)
    out = torch.empty((64, 9), dtype=torch.int32, device=DEV)
    a = tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 7, 0, 8, na, out)
    ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    for (B, L, ragged, seed) in ((37, 700, True, 3), (256, 4096, False, 11)):
        ctx, offs = synth.make_contexts(B=B, L=L, seed=seed, ragged=ragged)
        opr, opl = oracle.lookup(ctx, offs, 1, 4, 5)
        c, o = torch.tensor(ctx, device=DEV), torch.tensor(offs, device=DEV)
        cl = torch.tensor(np.diff(offs).astype(np.int32), device=DEV)
        pr = torch.full((B, 5), -7, dtype=torch.int32, device=DEV)
        pl = torch.full((B,), -7, dtype=torch.int32, device=DEV)
        alpha = torch.full((1,), 0.7, dtype=torch.float64, device=DEV)
        st = torch.zeros(1, dtype=torch.int32, device=DEV)
        for mode in ("eager", "graph"):
            pr.fill_(-7)
            pl.fill_(-7)
            g = torch.cuda.CUDAGraph() if mode == "graph" else None
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                ctxm = torch.cuda.graph(g, stream=side) if g is not None else torch.cuda.stream(side)
                with ctxm:
                    for rep in range(2):
                        tsv._check(tsv.lib().tsv_verify_accept(tsv.ctypes.byref(a), tsv._stream(None)))
                        tsv.tsv_propose_lookup(c, o, 1, 4, 5, proposals=pr, proposal_len=pl, device_status=st,
                                               flags=tsv.LOOKUP_INPUTS_READY)
                        tsv.tsv_goodput_choose_k(alpha, cl, pl, 5, tsv.POLICY_PLD, synth.SPEC_DESK_TARGET,
                                                 synth.SPEC_DESK_DRAFT, 0.05)
            torch.cuda.current_stream().wait_stream(side)
            if g is not None:
                pr.fill_(-7)
                pl.fill_(-7)
                g.replay()
            torch.cuda.synchronize()
            assert (_np(pl) == opl).all() and (_np(pr) == opr).all(), mode
            assert int(st.item()) == 0


def test_lookup_inputs_ready_bad_context_status(tsv):
    # the deferred status store: decreasing offsets still flag BAD_CONTEXT with the flag set
    ctx = torch.arange(64, dtype=torch.int32, device=DEV) % 7
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    pr, pl = tsv.tsv_propose_lookup(ctx, torch.tensor([0, 40, 20, 64], dtype=torch.int32, device=DEV), 1, 3, 4,
                                    device_status=st, flags=tsv.LOOKUP_INPUTS_READY)
    torch.cuda.synchronize()
    assert int(st.item()) == tsv.DEVSTATUS_BAD_CONTEXT and int(pl[1].item()) == 0 and (_np(pr)[1] == -1).all()


def test_lookup_config1(tsv):
    ctx, offs = synth.make_contexts(B=4, L=512, seed=1)
    plen = assert_lookup_parity(tsv, ctx, offs, 3, 3, 5)
    assert plen.sum() > 0


@pytest.mark.parametrize("n_min,n_max", [(1, 1), (2, 2), (3, 3), (4, 4), (1, 4)])
def test_lookup_config3(tsv, n_min, n_max):
    ctx, offs = synth.make_contexts(B=256, L=4096, seed=3)
    assert_lookup_parity(tsv, ctx, offs, n_min, n_max, 5)


def test_lookup_ragged_edges(tsv):
    rng = np.random.Generator(np.random.PCG64(7))
    ctxs = [rng.integers(0, A, L).astype(np.int32) for L in range(0, 60) for A in (1, 2, 4)]
    offs = np.zeros(len(ctxs) + 1, np.int32)
    offs[1:] = np.cumsum([len(c) for c in ctxs])
    flat = np.concatenate(ctxs)
    for (a, b, K) in [(1, 4, 5), (2, 3, 1), (1, 8, 15), (5, 5, 3)]:
        assert_lookup_parity(tsv, flat, offs, a, b, K)


def test_lookup_long_unstaged_and_unaligned(tsv):
    # 20000-token contexts exceed the shared-memory stage; odd offsets misalign the TMA copy
    ctx, offs = synth.make_contexts(B=6, L=20000, seed=9, ragged=True)
    assert_lookup_parity(tsv, ctx, offs, 1, 4, 5)
    ctx, offs = synth.make_contexts(B=33, L=3001, seed=10, ragged=True)
    assert_lookup_parity(tsv, ctx, offs, 2, 4, 7)


@pytest.mark.parametrize("n_min,n_max", [(1, 5), (3, 9), (1, 64), (64, 64)])
def test_lookup_long_ngrams(tsv, n_min, n_max):
    # periodic contexts with a small alphabet: suffix matches far longer than 4 tokens
    # exercise the walk beyond the branch-free 4-token window
    rng = np.random.Generator(np.random.PCG64(n_max))
    ctxs = []
    for b in range(40):
        period = int(rng.integers(1, 90))
        L = int(rng.integers(0, 700))
        base = rng.integers(0, 3, period).astype(np.int32)
        c = np.resize(base, L)
        if L and b % 3 == 0:
            c[rng.integers(0, L, 1 + L // 50)] = rng.integers(0, 3)  # break some repeats
        ctxs.append(c.astype(np.int32))
    offs = np.zeros(len(ctxs) + 1, np.int32)
    offs[1:] = np.cumsum([len(c) for c in ctxs])
    assert_lookup_parity(tsv, np.concatenate(ctxs), offs, n_min, n_max, 15)


# --------------------------------------------------------------------------- goodput
PROFILES = [(synth.SPEC_DESK_TARGET, synth.SPEC_DESK_DRAFT), (synth.H100_CASE_TARGET, synth.H100_CASE_DRAFT)]


def gpu_choose_k(tsv, alpha, ctx_len, cap, k_max, policy, target, draft, pld=0.0, kv=-1):
    a = torch.tensor(np.atleast_1d(np.asarray(alpha, np.float64)), device=DEV)
    cl = torch.tensor(np.asarray(ctx_len, np.int32), device=DEV)
    cp = torch.tensor(np.asarray(cap, np.int32), device=DEV)
    kpr = torch.empty_like(cp)
    k, g, kpr = tsv.tsv_goodput_choose_k(a, cl, cp, k_max, policy, target, draft, pld, kv,
                                         alpha_per_request=np.ndim(alpha) > 0, k_per_request=kpr)
    torch.cuda.synchronize()
    return int(k.item()), _np(g), _np(kpr)


def test_choose_k_config5_sweep(tsv):
    # batch 1-512 x alpha 0.3-0.9 x K=8, both latency profiles; bitwise k and goodput
    n = 0
    for target, draft in PROFILES:
        for B in list(range(1, 65)) + [96, 128, 200, 256, 300, 384, 511, 512]:
            ctx, cap = synth.make_goodput_instance(B, 8, seed=B)
            for a in (0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9):
                ok, og = oracle.choose_k(a, ctx, cap, 8, oracle.POLICY_DRAFT, target, draft)
                gk, gg, kpr = gpu_choose_k(tsv, a, ctx, cap, 8, 0, target, draft)
                assert gk == ok and (gg.view(np.uint64) == og.view(np.uint64)).all(), (B, a)
                assert (kpr == np.minimum(ok, cap)).all()
                n += 1
    assert n > 1000


def test_choose_k_pld_per_request_oom(tsv):
    rng = np.random.Generator(np.random.PCG64(3))
    for trial in range(60):
        B = int(rng.integers(1, 300))
        ctx, _ = synth.make_goodput_instance(B, 5, seed=trial)
        cap = rng.integers(0, 6, B).astype(np.int32)
        alpha = rng.uniform(0, 1, B)
        kv = int(rng.integers(-1, 4 * B))
        for pol in (0, 1):
            ok, og = oracle.choose_k(alpha, ctx, cap, 5, pol, synth.SPEC_DESK_TARGET,
                                     synth.SPEC_DESK_DRAFT, pld_cost_ms=0.05, kv_free_slots=kv)
            gk, gg, _ = gpu_choose_k(tsv, alpha, ctx, cap, 5, pol, synth.SPEC_DESK_TARGET,
                                     synth.SPEC_DESK_DRAFT, 0.05, kv)
            assert gk == ok and (gg.view(np.uint64) == og.view(np.uint64)).all()


def test_update_parity(tsv):
    rng = np.random.Generator(np.random.PCG64(4))
    for trial in range(40):
        B = int(rng.integers(1, 600))
        ks = rng.integers(0, 9, B)
        m = np.minimum(rng.geometric(0.3, B) - 1, ks).astype(np.int32)
        m[rng.random(B) < 0.02] = -1
        ro = np.zeros(B + 1, np.int32); ro[1:] = np.cumsum(ks + 1)
        for est in (0, 1):
            for per in (False, True):
                a0 = rng.uniform(0, 1, B) if per else float(rng.uniform(0, 1))
                want = oracle.update(a0, m, ro, decay=0.9, estimator=est)
                a = torch.tensor(np.atleast_1d(a0), dtype=torch.float64, device=DEV)
                tsv.tsv_update_acceptance(a, torch.tensor(m, device=DEV), torch.tensor(ro, device=DEV),
                                          0.9, est, per_request=per)
                got = _np(a)
                assert (got.view(np.uint64) == np.atleast_1d(want).view(np.uint64)).all()


# ------------------------------------------------------- request-sharded goodput / update (8e)
def _random_partition(rng, B, G):
    """G disjoint request subsets (some possibly empty), contiguous or scattered."""
    if rng.random() < 0.5:
        cuts = np.sort(rng.integers(0, B + 1, G - 1))
        bounds = np.concatenate([[0], cuts, [B]])
        return [np.arange(bounds[g], bounds[g + 1]) for g in range(G)]
    owner = rng.integers(0, G, B)
    return [np.flatnonzero(owner == g) for g in range(G)]


def test_goodput_sharded_sums_equal_oracle(tsv):
    # each "rank" reduces its own requests; the element-wise sum of the partials, finalized,
    # must give the oracle's k* and goodput bit for bit for any partition (exact int64 sums)
    rng = np.random.Generator(np.random.PCG64(8))
    for trial in range(60):
        B = int(rng.integers(1, 400))
        K = int(rng.integers(1, 9))
        ctx, _ = synth.make_goodput_instance(B, K, seed=100 + trial)
        cap = rng.integers(0, K + 1, B).astype(np.int32)
        per = trial % 2 == 1
        alpha = rng.uniform(0, 1, B) if per else float(rng.uniform(0.05, 0.95))
        kv = int(rng.integers(-1, 3 * B)) if trial % 3 == 0 else -1
        pol = trial % 2
        target, draft = PROFILES[trial % 2]
        ok, og = oracle.choose_k(alpha, ctx, cap, K, pol, target, draft, pld_cost_ms=0.05, kv_free_slots=kv)
        G = int(rng.integers(1, 9))
        parts = _random_partition(rng, B, G)
        total = torch.zeros(tsv.gp_sums_len(K), dtype=torch.int64, device=DEV)
        a_all = np.atleast_1d(np.asarray(alpha, np.float64))
        for idx in parts:
            a = torch.tensor(a_all[idx] if per else a_all, device=DEV)
            c = torch.tensor(ctx[idx], device=DEV)
            cp = torch.tensor(cap[idx], device=DEV)
            total += tsv.tsv_goodput_partial(a, c, cp, K, alpha_per_request=per)
        kpr_parts = []
        for idx in parts:  # every rank finalizes the same global sums; k_i for its own requests
            cp = torch.tensor(cap[idx], device=DEV)
            kpr = torch.empty_like(cp)
            k, g, _ = tsv.tsv_goodput_finalize(total, K, pol, target, draft, 0.05, kv, cap=cp, k_per_request=kpr)
            torch.cuda.synchronize()
            assert int(k.item()) == ok, (trial, G)
            assert (_np(g).view(np.uint64) == og.view(np.uint64)).all(), trial
            kpr_parts.append((idx, _np(kpr)))
        for idx, kp in kpr_parts:
            assert (kp == np.maximum(np.minimum(ok, cap[idx]), 0)).all()


def test_goodput_histogram_sums_equal_per_request_sums(tsv):
    # a global alpha takes the histogram path (sums from the counts of clamp(cap_i, 0, K)); the same
    # alpha given per request takes the per-request path: the exact int64 sums must be identical,
    # including K = 0, negative caps and caps above K (every word of the partial: L, N, sum ctx_len,
    # sum ctx_len over cap > 0, #{cap > 0}, B)
    rng = np.random.Generator(np.random.PCG64(12))
    for trial in range(40):
        B = int(rng.integers(1, 700))
        K = int(rng.integers(0, 9)) if trial % 4 else 0
        ctx = rng.integers(0, 5000, B).astype(np.int32)
        cap = rng.integers(-2, K + 4, B).astype(np.int32)
        a = float(rng.uniform(0, 1))
        c, cp = torch.tensor(ctx, device=DEV), torch.tensor(cap, device=DEV)
        hist = tsv.tsv_goodput_partial(torch.tensor([a], dtype=torch.float64, device=DEV), c, cp, K,
                                       alpha_per_request=False)
        per = tsv.tsv_goodput_partial(torch.full((B,), a, dtype=torch.float64, device=DEV), c, cp, K,
                                      alpha_per_request=True)
        torch.cuda.synchronize()
        assert torch.equal(hist, per), (trial, K, _np(hist), _np(per))
        capc = np.maximum(cap, 0).astype(np.int32)  # the oracle's caps are counts (>= 0)
        for pol in (0, 1):
            target, draft = PROFILES[pol]
            ok, og = oracle.choose_k(a, ctx, capc, K, pol, target, draft, pld_cost_ms=0.05)
            k, g, _ = tsv.tsv_goodput_choose_k(torch.tensor([a], dtype=torch.float64, device=DEV), c,
                                               torch.tensor(capc, device=DEV), K, pol, target, draft, 0.05)
            torch.cuda.synchronize()
            assert int(k.item()) == ok and (_np(g).view(np.uint64) == og.view(np.uint64)).all(), (trial, K, pol)


def test_update_sharded_sums_equal_oracle(tsv):
    rng = np.random.Generator(np.random.PCG64(9))
    for trial in range(40):
        B = int(rng.integers(1, 500))
        ks = rng.integers(0, 9, B)
        m = np.minimum(rng.geometric(0.3, B) - 1, ks).astype(np.int32)
        m[rng.random(B) < 0.02] = -1
        est = trial % 2
        a0 = float(rng.uniform(0, 1))
        want = oracle.update(a0, m, np.concatenate([[0], np.cumsum(ks + 1)]).astype(np.int32), 0.9, est)
        total = torch.zeros(2, dtype=torch.int64, device=DEV)
        for idx in _random_partition(rng, B, int(rng.integers(1, 9))):
            ro = np.zeros(len(idx) + 1, np.int32)
            ro[1:] = np.cumsum(ks[idx] + 1)
            total += tsv.tsv_update_partial(torch.tensor(m[idx], device=DEV), torch.tensor(ro, device=DEV), est)
        a = torch.tensor([a0], dtype=torch.float64, device=DEV)
        tsv.tsv_update_finalize(a, total, 0.9)
        assert (_np(a).view(np.uint64) == np.atleast_1d(want).view(np.uint64)).all()


def test_p2p_allreduce_loopback_streams(tsv):
    # G virtual ranks on one device, each on its own stream (the kernels run concurrently and poll
    # each other's LL words); exact int64 sums incl. wrap-around, three calls (both slot parities)
    rng = np.random.Generator(np.random.PCG64(12))
    for G in (1, 2, 4, 8):
        lb = tsv.P2PLoopback(G, 8)
        try:
            streams = [torch.cuda.Stream() for _ in range(G)]
            for call in range(3):
                n = int(rng.integers(1, 65))
                vals = rng.integers(-2 ** 62, 2 ** 62, (G, n), dtype=np.int64)
                vals[:, 0] = 2 ** 62  # sum wraps modulo 2^64 like the NCCL int64 sum
                data = [torch.tensor(vals[g], device=DEV) for g in range(G)]
                st = torch.zeros(1, dtype=torch.int32, device=DEV)
                torch.cuda.synchronize()
                for g in range(G):
                    tsv._check(tsv.lib().tsv_allreduce_i64_p2p(data[g].data_ptr(), n, lb.handles[g], st.data_ptr(),
                                                               streams[g].cuda_stream))
                torch.cuda.synchronize()
                want = vals.astype(np.uint64).sum(axis=0).view(np.int64)
                for g in range(G):
                    assert (_np(data[g]) == want).all(), (G, call, g)
                assert int(st.item()) == 0
        finally:
            lb.close()


def test_sharded_goodput_and_update_nccl_world1(tsv):
    # the NCCL plumbing (partial -> ncclAllReduce -> finalize) on a one-rank communicator
    comm = tsv.Comm(0, 1)
    try:
        B, K = 300, 5
        ctx, _ = synth.make_goodput_instance(B, K, seed=5)
        cap = np.random.Generator(np.random.PCG64(5)).integers(0, K + 1, B).astype(np.int32)
        for pol in (0, 1):
            ok, og = oracle.choose_k(0.7, ctx, cap, K, pol, synth.SPEC_DESK_TARGET, synth.SPEC_DESK_DRAFT,
                                     pld_cost_ms=0.05)
            a = torch.tensor([0.7], dtype=torch.float64, device=DEV)
            k, g, _ = tsv.tsv_goodput_choose_k_sharded(a, torch.tensor(ctx, device=DEV),
                                                       torch.tensor(cap, device=DEV), K, pol,
                                                       synth.SPEC_DESK_TARGET, comm, synth.SPEC_DESK_DRAFT, 0.05)
            torch.cuda.synchronize()
            assert int(k.item()) == ok and (_np(g).view(np.uint64) == og.view(np.uint64)).all()
        ks = np.full(B, K)
        m = np.minimum(np.arange(B) % 7, K).astype(np.int32)
        ro = np.concatenate([[0], np.cumsum(ks + 1)]).astype(np.int32)
        want = oracle.update(0.5, m, ro, 0.9, 0)
        a = torch.tensor([0.5], dtype=torch.float64, device=DEV)
        tsv.tsv_update_acceptance_sharded(a, torch.tensor(m, device=DEV), torch.tensor(ro, device=DEV), comm)
        assert (_np(a).view(np.uint64) == np.atleast_1d(want).view(np.uint64)).all()
    finally:
        comm.close()


# ------------------------------------------------------------------- fused entry points
def test_fused_lookup_choose_k_equals_separate(tsv):
    ctx, offs = synth.make_contexts(B=200, L=2048, seed=21, ragged=True)
    c, o = torch.tensor(ctx, device=DEV), torch.tensor(offs, device=DEV)
    ctx_len = torch.tensor(np.diff(offs).astype(np.int32), device=DEV)
    counter = tsv.lookup_choose_scratch(DEV)
    for a0 in (0.3, 0.7, 0.95):
        alpha = torch.tensor([a0], dtype=torch.float64, device=DEV)
        pr, pl = tsv.tsv_propose_lookup(c, o, 1, 4, 5)
        k, g, kpr = tsv.tsv_goodput_choose_k(alpha, ctx_len, pl, 5, tsv.POLICY_PLD, synth.SPEC_DESK_TARGET,
                                             synth.SPEC_DESK_DRAFT, 0.05, k_per_request=torch.empty_like(pl))
        kpr2 = torch.empty_like(pl)
        pr2, pl2, k2, g2 = tsv.tsv_propose_lookup_choose_k(c, o, 1, 4, 5, alpha, ctx_len, synth.SPEC_DESK_TARGET,
                                                           0.05, counter, k_per_request=kpr2)
        torch.cuda.synchronize()
        assert torch.equal(pr, pr2) and torch.equal(pl, pl2) and torch.equal(k, k2)
        assert torch.equal(g.view(torch.int64), g2.view(torch.int64)) and torch.equal(kpr, kpr2)
        assert int(counter.abs().sum().item()) == 0  # scratch left zero
        ok, og = oracle.choose_k(a0, np.diff(offs).astype(np.int32), _np(pl), 5, oracle.POLICY_PLD,
                                 synth.SPEC_DESK_TARGET, synth.SPEC_DESK_DRAFT, pld_cost_ms=0.05)
        assert int(k2.item()) == ok


def test_meta_ready_flag_same_outputs(tsv):
    # TSV_VERIFY_META_READY only moves the scan's first loads before its grid-dependency wait
    vb = synth.make_verify_batch(B=200, V=32000, k_max=8, lam=0.6, seed=31)
    ona, oout, _ = oracle_verify(vb, 3, 4)
    for flags in (tsv.VERIFY_META_READY, tsv.VERIFY_META_READY | tsv.VERIFY_NO_PRUNE):
        na, out, st = gpu_verify(tsv, vb, 3, 4, flags=flags)
        assert (na == ona).all() and (out == oout).all() and st == 0


def test_early_trigger_followed_by_dependent_kernels(tsv):
    # TSV_VERIFY_EARLY_TRIGGER: the kernel after the call may launch while the race runs; kernels that
    # read the call's outputs only after their own grid-dependency wait (the alpha update, the next
    # verify's scan for p / q and its workspace writes) still see them complete.  Three verify calls with
    # the flag, each followed by the standalone update, in one graph: every output equals the oracle
    vb = synth.make_verify_batch(B=200, V=32000, k_max=8, lam=0.6, seed=41).to(DEV)
    na = torch.empty(200, dtype=torch.int32, device=DEV)
    out = torch.empty((200, 9), dtype=torch.int32, device=DEV)
    alpha = torch.full((1,), 0.7, dtype=torch.float64, device=DEV)
    args = [tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 9, t, 8, na, out,
                                 flags=tsv.VERIFY_EARLY_TRIGGER | tsv.VERIFY_META_READY) for t in range(3)]
    ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(args[0]), DEV)
    for a in args:
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    outs = [torch.empty_like(out) for _ in range(3)]
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        tsv._check(tsv.lib().tsv_verify_accept(tsv.ctypes.byref(args[0]), tsv._stream(side)))  # warm-up
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=side):
            for t, a in enumerate(args):
                tsv._check(tsv.lib().tsv_verify_accept(tsv.ctypes.byref(a), tsv._stream(side)))
                tsv.tsv_update_acceptance(alpha, na, vb.row_offsets, 0.9, stream=side)
                outs[t].copy_(out)
    torch.cuda.current_stream().wait_stream(side)
    alpha.fill_(0.7)
    g.replay()
    torch.cuda.synchronize()
    h = synth.make_verify_batch(B=200, V=32000, k_max=8, lam=0.6, seed=41)
    a_ref = 0.7
    for t in range(3):
        ona, oout, _ = oracle_verify(h, 9, t)
        assert (_np(outs[t]) == oout).all(), t
        a_ref = oracle.update(a_ref, ona, _np(h.row_offsets), decay=0.9)
    assert float(alpha.item()) == a_ref


def test_alpha_ready_word_protocol(tsv):
    # tsv_verify_accept_update_ex: the word is reset by the call's first kernel and set to 1 once alpha is
    # written (global and per-request alpha); the fused lookup + choose-k waiting on it reads that alpha
    vb = synth.make_verify_batch(B=64, V=32000, k_max=8, lam=0.7, seed=43).to(DEV)
    h = synth.make_verify_batch(B=64, V=32000, k_max=8, lam=0.7, seed=43)
    ona, _, _ = oracle_verify(h, 3, 1)
    for per in (False, True):
        na = torch.empty(64, dtype=torch.int32, device=DEV)
        out = torch.empty((64, 9), dtype=torch.int32, device=DEV)
        a = tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 3, 1, 8, na, out)
        ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
        alpha = torch.full((64 if per else 1,), 0.7, dtype=torch.float64, device=DEV)
        ready = torch.full((1,), 7, dtype=torch.int32, device=DEV)
        tsv._check(tsv.lib().tsv_verify_accept_update_ex(tsv.ctypes.byref(a), alpha.data_ptr(), 1 if per else 0, 0.9,
                                                         tsv.EST_TESTED, ready.data_ptr(), tsv._stream(None)))
        torch.cuda.synchronize()
        assert int(ready.item()) == 1
        want = oracle.update(np.full(64, 0.7) if per else 0.7, ona, _np(h.row_offsets), decay=0.9)
        assert np.array_equal(_np(alpha), np.atleast_1d(want))


def test_alpha_ready_wait_times_out_without_producer(tsv):
    # a fused lookup + choose-k told to wait for alpha_ready that nobody sets gives up after the bounded
    # wait (TSV_DEVSTATUS_WAIT_TIMEOUT) instead of hanging; its outputs still follow the alpha it then reads
    ctx, offs = synth.make_contexts(B=8, L=256, seed=9)
    c, o = torch.tensor(ctx, device=DEV), torch.tensor(offs, device=DEV)
    cl = torch.tensor(np.diff(offs).astype(np.int32), device=DEV)
    alpha = torch.full((1,), 0.6, dtype=torch.float64, device=DEV)
    ready = torch.zeros(1, dtype=torch.int32, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    counter = tsv.lookup_choose_scratch(DEV)
    pr, pl, k, g = tsv.tsv_propose_lookup_choose_k(c, o, 1, 4, 5, alpha, cl, synth.SPEC_DESK_TARGET, 0.05, counter,
                                                   device_status=st, flags=tsv.LOOKUP_INPUTS_READY, alpha_ready=ready)
    torch.cuda.synchronize()
    assert int(st.item()) & tsv.DEVSTATUS_WAIT_TIMEOUT
    opr, opl = oracle.lookup(ctx, offs, 1, 4, 5)
    ok, _ = oracle.choose_k(0.6, np.diff(offs).astype(np.int32), opl, 5, oracle.POLICY_PLD, synth.SPEC_DESK_TARGET,
                            synth.SPEC_DESK_DRAFT, pld_cost_ms=0.05)
    assert (_np(pl) == opl).all() and int(k.item()) == ok


@pytest.mark.parametrize("chunk", [0, 128])
@pytest.mark.parametrize("est", [0, 1])  # TESTED (default), PROPOSED
def test_fused_verify_update_equals_separate(tsv, est, chunk):
    # the fused update runs beside the race: on the race grid's item-less last warp (chunk 0: 4608 work items
    # for 4736 warps) or as an extra CTA (chunk 128: 64000 items, every warp busy).  Same alpha bits as the
    # separate call either way.
    vb = synth.make_verify_batch(B=256, V=32000, k_max=8, lam=0.7, seed=22).to(DEV)
    for per in (False, True):
        na = torch.empty(256, dtype=torch.int32, device=DEV)
        out = torch.empty((256, 9), dtype=torch.int32, device=DEV)
        a = tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 7, 3, 8, na, out,
                                 chunk=chunk)
        ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), DEV)
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
        a0 = torch.rand(256 if per else 1, dtype=torch.float64, device=DEV, generator=torch.Generator(DEV).manual_seed(1))
        alpha1 = a0.clone()
        tsv._check(tsv.lib().tsv_verify_accept(tsv.ctypes.byref(a), tsv._stream(None)))
        tsv.tsv_update_acceptance(alpha1, na, vb.row_offsets, 0.9, estimator=est, per_request=per)
        out1, na1 = out.clone(), na.clone()
        alpha2 = a0.clone()
        tsv.tsv_verify_accept_update(a, alpha2, 0.9, estimator=est, per_request=per)
        torch.cuda.synchronize()
        assert torch.equal(out1, out) and torch.equal(na1, na)
        assert torch.equal(alpha1.view(torch.int64), alpha2.view(torch.int64))


# ------------------------------------------------------------------- whole step in a graph
@pytest.mark.parametrize("fused", [False, True])
def test_step_graph_capture_matches_eager(tsv, fused):
    from paper_2406_14066_b200.step import SpecStep, StepInputs
    inp = synth.make_step_inputs(B=64, V=32000, L=1024, k_max=8, seed=20, device=DEV)
    st = SpecStep(inp, fused=fused)
    st.run(step=0)
    torch.cuda.synchronize()
    eager = {k: v.clone() for k, v in st.outputs().items()}
    st2 = SpecStep(inp, fused=not fused)
    st2.capture(steps=[0])
    st2.replay()
    torch.cuda.synchronize()
    for k, v in st2.outputs().items():
        assert torch.equal(v, eager[k]), k


@pytest.mark.slow
def test_bench_step_full_size_equals_oracle(tsv):
    # the bench's step at its full size and in the launch configuration bench.py times (B = 256,
    # V = 32000, k in 0..8, L = 4096, n 1-4, K = 5; two rotation sets; four consecutive steps in one
    # CUDA graph, TSV_LOOKUP_INPUTS_READY and TSV_VERIFY_META_READY set, alpha carried from step to
    # step) against the oracle's composition of Listing 1: lookup -> choose-k -> verify -> update
    from paper_2406_14066_b200.step import SpecStep
    inp = synth.make_step_inputs(B=256, V=32000, L=4096, k_max=8, seed=240614066, device=DEV, sets=2)
    st = SpecStep(inp)
    steps = [0, 1, 2, 3]
    st.capture(steps)
    st.reset_state()
    st.replay()
    torch.cuda.synchronize()
    alpha = 0.7
    for t in steps:
        s = t % inp.sets
        ctx, offs = _np(inp.ctx[s]), _np(inp.ctx_offsets[s])
        opr, opl = oracle.lookup(ctx, offs, 1, 4, 5)
        ok, og = oracle.choose_k(alpha, np.diff(offs).astype(np.int32), opl, 5, oracle.POLICY_PLD,
                                 synth.SPEC_DESK_TARGET, synth.SPEC_DESK_DRAFT, pld_cost_ms=0.05)
        vb = inp.verify[s]
        ona, oout, _ = oracle.verify(_np(vb.p), _np(vb.q), _np(vb.row_offsets), _np(vb.draft_tokens),
                                     _np(vb.request_ids).view(np.uint32), inp.seed, t, 8, vocab=32000)
        alpha = oracle.update(alpha, ona, _np(vb.row_offsets), decay=0.9)
    # the graph's buffers hold the last step's outputs (and alpha after all four updates)
    assert (_np(st.proposal_len) == opl).all() and (_np(st.proposals) == opr).all()
    assert int(st.k_star.item()) == ok
    assert (_np(st.goodput).view(np.uint64) == og.view(np.uint64)).all()
    assert (_np(st.num_accepted) == ona).all() and (_np(st.out_tokens) == oout).all()
    assert float(st.alpha.item()) == alpha and int(st.status.item()) == 0


@pytest.mark.parametrize("fused", [False, True])
def test_step_lookup_ready_multi_step_graph_matches_eager(tsv, fused):
    # three consecutive steps in one graph with TSV_LOOKUP_INPUTS_READY (the lookup of step t+1 -- and,
    # fused, its ArgMaxGoodput over alpha from step t's update -- runs while step t's emit drains) equal
    # three eager steps of the separate calls without the flag (alpha carried across steps)
    from paper_2406_14066_b200.step import SpecStep
    inp = synth.make_step_inputs(B=96, V=32000, L=2048, k_max=8, seed=21, device=DEV, sets=2)
    st = SpecStep(inp, lookup_ready=False)
    for t in range(3):
        st.run(step=t)
    torch.cuda.synchronize()
    eager = {k: v.clone() for k, v in st.outputs().items()}
    st2 = SpecStep(inp, lookup_ready=True, fused=fused)
    st2.capture(steps=[0, 1, 2])
    st2.replay()
    torch.cuda.synchronize()
    for k, v in st2.outputs().items():
        assert torch.equal(v, eager[k]), k


# ------------------------------------------------------------------- greedy verify (NEXT 2)
def assert_greedy_parity(tsv, p, ro, drafts, k_max, vocab=None, chunk=0):
    ona, oout, ost = oracle.verify_greedy(p, ro, drafts, k_max, vocab=vocab)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    dt = torch.tensor(drafts if len(drafts) else np.zeros(0, np.int32), dtype=torch.int32, device=DEV)
    na, out = tsv.tsv_verify_greedy(torch.tensor(p, device=DEV), torch.tensor(ro, device=DEV), dt, k_max,
                                    device_status=st, vocab=vocab, chunk=chunk)
    torch.cuda.synchronize()
    assert (_np(na) == ona).all() and (_np(out) == oout).all()
    assert int(st.item()) == ost
    return ona


def _greedy_batch(B, V, k_max, seed, accept=0.7, ld=None, ties=False):
    rng = np.random.Generator(np.random.PCG64(seed))
    ks = rng.integers(0, k_max + 1, B)
    ro = np.zeros(B + 1, np.int32)
    ro[1:] = np.cumsum(ks + 1)
    R = int(ro[-1])
    ld = (V + 3) // 4 * 4 if ld is None else ld  # rows padded to a multiple of 4 (tsv_verify_args.ld)
    if ties:
        p = rng.integers(0, 5, (R, ld)).astype(np.float32)
    else:
        p = rng.standard_normal((R, ld)).astype(np.float32)
    am = p[:, :V].argmax(axis=1)
    drafts = []
    for i in range(B):
        for j in range(ks[i]):
            r = ro[i] + j
            drafts.append(int(am[r]) if rng.random() < accept else int(rng.integers(0, V)))
    return p, ro, np.array(drafts, np.int32)


@pytest.mark.parametrize("B,V,k_max", [(4, 32000, 4), (256, 32000, 8), (37, 4099, 15), (9, 13, 3), (5, 1, 2)])
def test_greedy_parity(tsv, B, V, k_max):
    p, ro, d = _greedy_batch(B, V, k_max, seed=B + V)
    na = assert_greedy_parity(tsv, p, ro, d, k_max, vocab=V)
    assert (na >= 0).all()


def test_greedy_ties_nan_padded_chunks(tsv):
    p, ro, d = _greedy_batch(50, 3000, 6, seed=3, ties=True, ld=3008)
    p[:, 3000:] = 1e30  # beyond vocab: never read
    for chunk in (0, 128, 640):
        assert_greedy_parity(tsv, p, ro, d, 6, vocab=3000, chunk=chunk)
    p2, ro2, d2 = _greedy_batch(20, 700, 4, seed=4)
    p2[::3, ::7] = np.nan
    p2[5] = np.nan                       # all-NaN row -> NO_WEIGHT if it is emitted
    p2[7] = -np.inf
    p2[9, :] = 0.0
    p2[9, 350] = -0.0
    assert_greedy_parity(tsv, p2, ro2, d2, 4)


def test_greedy_bad_tokens(tsv):
    p, ro, d = _greedy_batch(12, 500, 3, seed=5)
    if len(d):
        d[0] = 500
    assert_greedy_parity(tsv, p, ro, d, 3)


# ------------------------------------------------------- fused softmax from logits (NEXT 1)
def test_softmax_rows_parity(tsv):
    rng = np.random.Generator(np.random.PCG64(51))
    # the row sums use the statistics pass's terms (one ex2.approx each): the bound is checked
    # on wide logit ranges (sigma 8-20, tau 0.5) as well as the synthetic recipe's sigma = 3
    for V, ld, tau, sigma in [(32000, 32000, 1.0, 3.0), (4099, 4100, 0.7, 2.0), (13, 16, 1.5, 8.0), (1, 4, 1.0, 1.0),
                              (128256, 128256, 1.0, 3.0), (32000, 32000, 0.5, 8.0), (5000, 5000, 1.0, 20.0)]:
        z = (rng.standard_normal((7, ld)) * sigma).astype(np.float32)
        z[0, : min(V - 1, 5)] = -np.inf  # -inf logits: probability 0 (a row keeps one finite logit)
        want = oracle.softmax_rows(z, tau, vocab=V)
        got = _np(tsv.tsv_softmax_rows(torch.tensor(z, device=DEV), tau, vocab=V))
        torch.cuda.synchronize()
        big = want > 1e-30
        rel = np.abs(got[big] - want[big]) / want[big]
        print(f"softmax rows V={V} tau={tau} sigma={sigma}: max relative error {rel.max():.3e}")
        assert rel.max() <= 1e-6, (V, tau, rel.max())
        assert (got[~big] <= 1e-30).all() and (got[:, V:] == 0).all()


def _race_scores(p_row, q_row, x_m, residual, seed, step, rid, m):
    """Oracle-side scores RN32(w / E(u)) of one raced row (diagnostics for near-tie listing)."""
    V = p_row.size
    if residual:
        w = (p_row - (q_row if q_row is not None else (np.arange(V) == x_m).astype(np.float32))).astype(np.float32)
        w = np.where(w > 0, w, 0).astype(np.float32)
    else:
        w = np.where(p_row > 0, p_row, 0).astype(np.float32)
    words = np.zeros(V, np.uint32)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for quad in range((V + 3) // 4):
        out = oracle.philox4x32_10([quad, (1 << 16) | m, rid, step], key)
        n = min(4, V - 4 * quad)
        words[4 * quad:4 * quad + n] = out[:n]
    E = _E_TABLE()[words & 0x7FFFFF]
    return np.where(w > 0, (w / E).astype(np.float32), -1.0).astype(np.float32)


_E_CACHE = []


def _E_TABLE():
    if not _E_CACHE:
        _E_CACHE.append(oracle.E_table())
    return _E_CACHE[0]


def near_tie_flips(vb, p, q, ona, oout, gna, gout, seed, step, tol=2e-6):
    """Requests whose GPU and oracle results differ, each classified: a flip is a near tie if
    the deciding comparison (acceptance u q vs p, or the race's top two scores) is within tol."""
    ro = _np(vb.row_offsets)
    dt = _np(vb.draft_tokens)
    rid = _np(vb.request_ids).view(np.uint32)
    flips = []
    for i in np.nonzero((ona != gna) | (oout != gout).any(1))[0]:
        r0, k = int(ro[i]), int(ro[i + 1] - ro[i] - 1)
        qb = r0 - int(i)
        reason = None
        m = int(min(ona[i], gna[i]))
        for j in range(m + 1 if m < k else k):  # acceptance decisions up to the first disagreement
            x = int(dt[qb + j])
            word = oracle.philox4x32_10([0, j, int(rid[i]), step], [seed & 0xFFFFFFFF, seed >> 32])[0]
            u = oracle.u_acc(int(word))
            uq = np.float32(u) * np.float32(q[qb + j, x] if q is not None else 1.0)
            if abs(float(uq) - float(p[r0 + j, x])) <= tol * max(float(p[r0 + j, x]), 1e-30):
                reason = f"accept j={j}: u*q={float(uq):.9g} vs p={float(p[r0 + j, x]):.9g}"
        if reason is None and ona[i] == gna[i]:
            mm = int(ona[i])
            sc = _race_scores(p[r0 + mm, :vb.vocab], None if (q is None or mm >= k) else q[qb + mm, :vb.vocab],
                              int(dt[qb + mm]) if mm < k else -1, mm < k, seed, step, int(rid[i]), mm)
            a, b = int(oout[i, mm]), int(gout[i, mm])
            if a >= 0 and b >= 0 and abs(float(sc[a]) - float(sc[b])) <= tol * float(max(sc[a], sc[b])):
                reason = f"race m={mm}: score[{a}]={float(sc[a]):.9g} vs score[{b}]={float(sc[b]):.9g}"
        flips.append((int(i), reason))
    return flips


@pytest.mark.parametrize("B,V,k_max,tau,dense_q", [(4, 32000, 4, 1.0, True), (128, 32000, 8, 1.0, True),
                                                   (64, 4099, 6, 0.8, True), (48, 32000, 5, 1.3, False)])
def test_verify_logits_parity(tsv, B, V, k_max, tau, dense_q):
    vb = synth.make_logits_batch(B=B, V=V, k_max=k_max, lam=0.7, seed=60 + B, dense_q=dense_q)
    seed, step = 240614066, 3
    zp, zq = _np(vb.p), _np(vb.q)
    p = oracle.softmax_rows(zp, tau, vocab=V)
    q = None if zq is None else oracle.softmax_rows(zq, tau, vocab=V)
    ona, oout, ost = oracle.verify(p, q, _np(vb.row_offsets), _np(vb.draft_tokens),
                                   _np(vb.request_ids).view(np.uint32), seed, step, k_max, vocab=V)
    g = vb.to(DEV)
    gna, gout = tsv.tsv_verify_accept_logits(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, seed, step,
                                             k_max, temperature=tau, vocab=V)
    torch.cuda.synchronize()
    gna, gout = _np(gna), _np(gout)
    flips = near_tie_flips(vb, p, q, ona, oout, gna, gout, seed, step)
    record_flips(dict(B=B, V=V, k_max=k_max, tau=tau, dense_q=dense_q, seed=seed, step=step), flips)
    assert all(reason is not None for _, reason in flips), flips
    assert len(flips) <= max(1, B // 64)


def record_flips(case, flips):
    """Every near-tie flip is listed (north_star): printed, and appended as one JSON line per case to
    gpurun_out/logits_flips.jsonl (the GPU run's artifact; the committed copy is under profiles/)."""
    import json
    for f in flips:
        print("near-tie flip:", case, f)
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "logits_flips.jsonl"), "a") as fh:
        fh.write(json.dumps({"case": case, "requests": case["B"], "flips": [{"request": i, "near_tie": r}
                                                                              for i, r in flips]}) + "\n")


@pytest.mark.slow
def test_verify_logits_parity_bench_size(tsv):
    # the bench's logits workload (B = 256, V = 32000, k in 0..8, tau = 1) at two Philox steps: every token
    # equal to the oracle's verify on the oracle's probabilities, or a listed near tie
    vb = synth.make_logits_batch(B=256, V=32000, k_max=8, lam=0.7, seed=240614066, dense_q=True)
    zp, zq = _np(vb.p), _np(vb.q)
    p, q = oracle.softmax_rows(zp, 1.0, vocab=32000), oracle.softmax_rows(zq, 1.0, vocab=32000)
    g = vb.to(DEV)
    for step in (0, 1):
        ona, oout, _ = oracle.verify(p, q, _np(vb.row_offsets), _np(vb.draft_tokens),
                                     _np(vb.request_ids).view(np.uint32), 240614066, step, 8, vocab=32000)
        gna, gout = tsv.tsv_verify_accept_logits(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, 240614066,
                                                 step, 8, temperature=1.0, vocab=32000)
        torch.cuda.synchronize()
        gna, gout = _np(gna), _np(gout)
        flips = near_tie_flips(vb, p, q, ona, oout, gna, gout, 240614066, step)
        record_flips(dict(B=256, V=32000, k_max=8, tau=1.0, dense_q=True, seed=240614066, step=step), flips)
        assert all(reason is not None for _, reason in flips), flips
        assert len(flips) <= 4


def test_verify_logits_prune_off_identical(tsv):
    vb = synth.make_logits_batch(B=32, V=4096, k_max=5, lam=0.6, seed=70).to(DEV)
    a = tsv.tsv_verify_accept_logits(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 9, 1, 5)
    b = tsv.tsv_verify_accept_logits(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, 9, 1, 5,
                                     flags=tsv.VERIFY_NO_PRUNE)
    torch.cuda.synchronize()
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()


# ------------------------------------------------------------------- zero-copy host inputs
def test_pinned_host_inputs_zero_copy(tsv):
    # p, q and the metadata left in pinned host memory: the kernels read them over PCIe (UVA)
    vb = synth.make_verify_batch(B=64, V=32000, k_max=8, lam=0.7, seed=26)
    ona, oout, _ = oracle_verify(vb, 7, 2)
    pin = lambda t: t.contiguous().pin_memory()
    na, out = tsv.tsv_verify_accept(pin(vb.p), pin(vb.q), pin(vb.row_offsets), pin(vb.draft_tokens),
                                    pin(vb.request_ids), 7, 2, 8,
                                    num_accepted=torch.empty(64, dtype=torch.int32, device=DEV),
                                    out_tokens=torch.empty((64, 9), dtype=torch.int32, device=DEV))
    torch.cuda.synchronize()
    assert (_np(na) == ona).all() and (_np(out) == oout).all()
    ctx, offs = synth.make_contexts(B=16, L=1024, seed=27)
    pr, pl = tsv.tsv_propose_lookup(pin(torch.tensor(ctx)), pin(torch.tensor(offs)), 1, 4, 5)
    opr, opl = oracle.lookup(ctx, offs, 1, 4, 5)
    assert (_np(pr) == opr).all() and (_np(pl) == opl).all()


# ------------------------------------------------------------------- randomised shape sweep
def test_random_shape_sweep(tsv):
    # 40 random (B, V, ld, k_max, lambda, dense/one-hot, chunk, seed, step) draws, bit-exact
    rng = np.random.Generator(np.random.PCG64(99))
    for trial in range(40):
        B = int(rng.integers(1, 80))
        V = int(rng.integers(1, 9000))
        ld = (V + 3) // 4 * 4 + 4 * int(rng.integers(0, 3))
        k_max = int(rng.integers(0, 16))
        dense = bool(rng.random() < 0.7)
        lam = float(rng.uniform(0.05, 0.99))
        chunk = int(rng.choice([0, 128, 512, 1536]))
        vb = synth.make_verify_batch(B=B, V=V, k_max=k_max, lam=lam, seed=1000 + trial, dense_q=dense, ld=ld)
        seed, step = int(rng.integers(0, 2 ** 63)), int(rng.integers(0, 2 ** 32))
        assert_verify_parity(tsv, vb, seed=seed, step=step, chunk=chunk)


# Shapes around the work-item and grid boundaries of the lazy race at the default chunk:
# one request, V at and around powers of two, V not a multiple of 4, more requests than SMs,
# Llama-3 vocabulary, thousands of short rows; pruned and unpruned.
@pytest.mark.parametrize("B,V,k_max,dense", [
    (1, 5, 3, True), (1, 8192, 8, True), (2, 8193, 8, False), (3, 16385, 4, True), (147, 100, 2, True),
    (149, 24577, 8, True), (300, 8191, 6, False), (257, 128256, 3, True), (4096, 64, 2, True),
    (4097, 64, 2, True)])
def test_race_shapes(tsv, B, V, k_max, dense):
    vb = synth.make_verify_batch(B=B, V=V, k_max=k_max, lam=0.7, seed=B * 131 + V, dense_q=dense)
    assert_verify_parity(tsv, vb, seed=B + V, step=B)
    assert_verify_parity(tsv, vb, seed=B + V, step=B, flags=tsv.VERIFY_NO_PRUNE)


def test_choose_k_batched_config5_sweep(tsv):
    # BASELINE config 5: batch 1-512 x alpha 0.3-0.9, K = 8, both policies, one launch per sweep
    for target, draft in PROFILES:
        for pol in (0, 1):
            Bs = list(range(1, 65)) + [96, 128, 200, 256, 300, 384, 511, 512]
            alphas = (0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9)
            ctxs, caps, offs, al, want_k, want_g = [], [], [0], [], [], []
            for B in Bs:
                ctx, cap = synth.make_goodput_instance(B, 8, seed=B)
                if pol == 1:
                    cap = np.random.Generator(np.random.PCG64(B)).integers(0, 9, B).astype(np.int32)
                for a in alphas:
                    ok, og = oracle.choose_k(a, ctx, cap, 8, pol, target, draft, pld_cost_ms=0.05)
                    ctxs.append(ctx)
                    caps.append(cap)
                    offs.append(offs[-1] + B)
                    al.append(a)
                    want_k.append(ok)
                    want_g.append(og)
            k, g = tsv.tsv_goodput_choose_k_batched(
                torch.tensor(al, dtype=torch.float64, device=DEV), torch.tensor(np.concatenate(ctxs), device=DEV),
                torch.tensor(np.concatenate(caps), device=DEV), torch.tensor(np.array(offs, np.int32), device=DEV),
                8, pol, target, draft, 0.05)
            torch.cuda.synchronize()
            assert (_np(k) == np.array(want_k)).all()
            assert (_np(g).view(np.uint64) == np.stack(want_g).view(np.uint64)).all()
