"""Worker of tests/test_gpu_dist_step.py (launched by torch.distributed.run, gloo, 2+ ranks).

One TurboSpec server over the ranks (request-sharded): every rank runs
SpecStep on its part of the batch with a P2PComm (peer-memory exchanges inside
tsv_goodput_choose_k_p2p and tsv_verify_accept_update_p2p), so alpha and k* are global.
Two partitions of the requests:
  strong  one B = 64 batch split by dist.partition_requests (what bench.py's "strong" times);
  weak    every rank generates its own B = 40 batch with global request ids rank*40 + i.
Rank 0 runs the oracle's step (lookup -> choose-k PLD -> verify -> update, oracle/) on the
union of the requests for the same step counters and checks every rank's k*, goodput bits,
alpha bits, proposals, k_i, accepted counts and emitted tokens -- eager steps, then the
same steps replayed from one captured CUDA graph.  Prints DIST-STEP-OK <rank> on success."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2406_14066_b200 import dist as pdist  # noqa: E402
from paper_2406_14066_b200 import tsv  # noqa: E402
from paper_2406_14066_b200.step import SpecStep, StepInputs  # noqa: E402

SEED = 77
STEPS = [0, 1, 2, 3]
K_MAX, V, L = 8, 8192, 1024


def oracle_steps(vb, ctx, offs, steps):
    """The oracle's decode steps on the whole batch: per step (k*, goodput, alpha after, proposals,
    lengths, k_i, accepted, tokens)."""
    p, q, ro = vb.p.numpy(), vb.q.numpy(), vb.row_offsets.numpy()
    d, rid = vb.draft_tokens.numpy(), vb.request_ids.numpy().view(np.uint32)
    ctx_len = np.diff(offs).astype(np.int32)
    alpha, res = 0.7, []
    for t in steps:
        pr, pl = oracle.lookup(ctx, offs, 1, 4, 5)
        k, g = oracle.choose_k(alpha, ctx_len, pl, 5, oracle.POLICY_PLD, synth.SPEC_DESK_TARGET,
                               synth.SPEC_DESK_DRAFT, pld_cost_ms=0.05)
        na, out, _ = oracle.verify(p, q, ro, d, rid, SEED, t, K_MAX)
        alpha = oracle.update(alpha, na, ro, decay=0.9)
        res.append((k, g, alpha, pr, pl, np.minimum(k, pl), na, out))
    return res


def concat_batches(parts):
    """Union of per-rank batches (rows concatenated in rank order; request ids already global)."""
    ro = [np.zeros(1, np.int64)]
    for vb in parts:
        ro.append(vb.row_offsets.numpy()[1:].astype(np.int64) + ro[-1][-1])
    return synth.VerifyBatch(torch.cat([vb.p for vb in parts]), torch.cat([vb.q for vb in parts]),
                             torch.tensor(np.concatenate(ro).astype(np.int32)),
                             torch.cat([vb.draft_tokens for vb in parts]), torch.cat([vb.request_ids for vb in parts]),
                             torch.cat([vb.k for vb in parts]), V, K_MAX)


def run_mode(mode, rank, world, dev):
    if mode == "strong":
        B = 64
        whole = synth.make_verify_batch(B=B, V=V, k_max=K_MAX, lam=0.7, seed=SEED)
        ctx, offs = synth.make_contexts(B=B, L=L, V=V, seed=SEED)
        lo, hi = pdist.partition_requests(whole.k.numpy(), world)[rank]
        g = whole.to(dev)
        p, q, ro, d, rid = pdist.request_slice(g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids, lo, hi)
        c, o = pdist.context_slice(torch.tensor(ctx, device=dev), torch.tensor(offs, device=dev), lo, hi)
        mine = (p, q, ro, d, rid)
        sel = np.arange(lo, hi)
    else:
        Br = 40
        parts = [synth.make_verify_batch(B=Br, V=V, k_max=K_MAX, lam=0.7, seed=SEED + 13 * r, request_id_base=r * Br)
                 for r in range(world)]
        ctxs = [synth.make_contexts(B=Br, L=L, V=V, seed=SEED + 13 * r) for r in range(world)]
        whole = concat_batches(parts)
        ctx = np.concatenate([c for c, _ in ctxs])
        offs = np.concatenate([[0]] + [o[1:] + r * Br * L for r, (_, o) in enumerate(ctxs)]).astype(np.int32)
        g = parts[rank].to(dev)
        mine = (g.p, g.q, g.row_offsets, g.draft_tokens, g.request_ids)
        c, o = torch.tensor(ctxs[rank][0], device=dev), torch.tensor(ctxs[rank][1], device=dev)
        sel = np.arange(rank * Br, (rank + 1) * Br)

    class VB:  # the arrays SpecStep reads
        pass
    vb = VB()
    vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids = mine
    inp = StepInputs([vb], [c.contiguous()], [o.contiguous()], [(o[1:] - o[:-1]).to(torch.int32).contiguous()], K_MAX,
                     seed=SEED)
    comm = tsv.P2PComm(rank, world, B_max=128)
    st = SpecStep(inp, device=dev, comm=comm)
    want = oracle_steps(whole, ctx, offs, STEPS) if rank == 0 else None
    ok = True

    def check(tag, outs):
        nonlocal ok
        gathered = [None] * world
        dist.all_gather_object(gathered, (sel, outs))
        if rank != 0:
            return
        for t_i, t in enumerate(STEPS):
            k, g_, alpha, pr, pl, kreq, na, out = want[t_i]
            for r, (sl, o_) in enumerate(gathered):
                rk, rg, ra, rpr, rpl, rkr, rna, rout, rst = o_[t_i]
                good = (rk == k and (rg.view(np.uint64) == g_.view(np.uint64)).all() and ra == alpha
                        and (rpr == pr[sl]).all() and (rpl == pl[sl]).all() and (rkr == kreq[sl]).all()
                        and (rna == na[sl]).all() and (rout == out[sl]).all() and rst == 0)
                if not good:
                    print(f"{mode} {tag} step {t} rank {r}: MISMATCH k {rk} vs {k}, alpha {ra} vs {alpha}, "
                          f"na {(rna != na[sl]).sum()} bad, status {rst}", flush=True)
                ok = ok and good
        print(f"{mode} {tag}: {'match' if ok else 'MISMATCH'}", flush=True)

    def snapshot():
        torch.cuda.synchronize()
        return (int(st.k_star.item()), st.goodput.cpu().numpy().copy(), float(st.alpha.item()),
                st.proposals.cpu().numpy().copy(), st.proposal_len.cpu().numpy().copy(), st.k_req.cpu().numpy().copy(),
                st.num_accepted.cpu().numpy().copy(), st.out_tokens.cpu().numpy().copy(), int(st.status.item()))

    st.reset_state()
    outs = []
    for t in STEPS:
        st.run(step=t)
        outs.append(snapshot())
    check("eager", outs)
    # the same steps as one CUDA graph per step (replayed in order; the exchange epochs live on the device)
    graphs = []
    for t in STEPS:
        st.capture([t])
        graphs.append(st.graph)
    dist.barrier()
    st.reset_state()
    outs = []
    for gph in graphs:
        gph.replay()
        outs.append(snapshot())
    check("graph", outs)
    dist.barrier()
    comm.close()
    return ok


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    ok = True
    for mode in ("strong", "weak"):
        ok = run_mode(mode, rank, world, dev) and ok
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    if int(flag.item()) == 1:
        print(f"DIST-STEP-OK {rank}", flush=True)
    sys.exit(0 if int(flag.item()) == 1 else 1)


if __name__ == "__main__":
    main()
