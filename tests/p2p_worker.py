"""Worker of test_p2p_vocab_shard_two_processes_ipc (launched by torch.distributed.run, 2 ranks).

Rank r runs on GPU r % device_count (two GPUs: a real NVLink peer mapping; one GPU: both ranks
share it); each holds one vocab shard of the same batch, maps the
other's symmetric buffer over CUDA IPC (tsv.P2PComm, handles exchanged over gloo) and runs
tsv_verify_accept_sharded_p2p for several steps, then the request-sharded global goodput and
alpha update over the same buffers; every result must equal the oracle on the whole batch."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2406_14066_b200 import tsv  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", rank % ndev)  # distinct GPUs when there are enough (NVLink), else shared
    torch.cuda.set_device(dev)
    vb = synth.make_verify_batch(B=48, V=32000, k_max=8, lam=0.7, seed=29)
    V, B = vb.vocab, vb.B
    Vs = V // world
    lo = rank * Vs
    g = vb.to(dev)
    p = g.p[:, lo:lo + Vs].contiguous()
    q = g.q[:, lo:lo + Vs].contiguous()
    comm = tsv.P2PComm(rank, world, B_max=64)
    na = torch.empty(B, dtype=torch.int32, device=dev)
    out = torch.empty((B, vb.k_max + 1), dtype=torch.int32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    ok = True
    for step in range(8):  # steps 0-3: LL keys kernel; steps 4-7: keys pushed by the race items (P2P_FUSED)
        fl = tsv.VERIFY_P2P_FUSED if step >= 4 else 0
        a = tsv.make_verify_args(p, q, g.row_offsets, g.draft_tokens, g.request_ids, 31, step, vb.k_max, na, out,
                                 device_status=st, vocab=Vs, vocab_offset=lo, vocab_global=V, flags=fl)
        ws = tsv.alloc_workspace(tsv.tsv_verify_workspace_size(a), dev)
        a.workspace = ws.data_ptr()
        a.workspace_bytes = ws.numel()
        tsv.tsv_verify_accept_sharded_p2p(a, comm)
        torch.cuda.synchronize()
        ona, oout, ost = oracle.verify(vb.p.numpy(), vb.q.numpy(), vb.row_offsets.numpy(), vb.draft_tokens.numpy(),
                                       vb.request_ids.numpy().view(np.uint32), 31, step, vb.k_max, vocab=V)
        good = (na.cpu().numpy() == ona).all() and (out.cpu().numpy() == oout).all() and int(st.item()) == ost
        print(f"rank {rank} step {step}: {'match' if good else 'MISMATCH'} status {int(st.item())}", flush=True)
        ok = ok and good
    # request-sharded global goodput and alpha update through the same buffers: rank r owns a
    # contiguous half of a B = 300 batch; k* / goodput / alpha must equal the oracle on the whole batch
    Bq, K = 300, 5
    ctx, _ = synth.make_goodput_instance(Bq, K, seed=31)
    cap = np.random.Generator(np.random.PCG64(31)).integers(0, K + 1, Bq).astype(np.int32)
    lo_r, hi_r = Bq * rank // world, Bq * (rank + 1) // world
    for pol in (0, 1):
        ok_k, og = oracle.choose_k(0.7, ctx, cap, K, pol, synth.SPEC_DESK_TARGET, synth.SPEC_DESK_DRAFT,
                                   pld_cost_ms=0.05)
        a = torch.tensor([0.7], dtype=torch.float64, device=dev)
        k, gp, _ = tsv.tsv_goodput_choose_k_sharded(a, torch.tensor(ctx[lo_r:hi_r], device=dev),
                                                    torch.tensor(cap[lo_r:hi_r], device=dev), K, pol,
                                                    synth.SPEC_DESK_TARGET, comm, synth.SPEC_DESK_DRAFT, 0.05)
        torch.cuda.synchronize()
        good = int(k.item()) == ok_k and (gp.cpu().numpy().view(np.uint64) == og.view(np.uint64)).all()
        print(f"rank {rank} goodput policy {pol}: {'match' if good else 'MISMATCH'}", flush=True)
        ok = ok and good
    ks = np.full(Bq, K)
    m = np.minimum(np.arange(Bq) % 7, K).astype(np.int32)
    want = oracle.update(0.5, m, np.concatenate([[0], np.cumsum(ks + 1)]).astype(np.int32), 0.9, 0)
    ro = np.concatenate([[0], np.cumsum(ks[lo_r:hi_r] + 1)]).astype(np.int32)
    a = torch.tensor([0.5], dtype=torch.float64, device=dev)
    tsv.tsv_update_acceptance_sharded(a, torch.tensor(m[lo_r:hi_r], device=dev), torch.tensor(ro, device=dev), comm)
    torch.cuda.synchronize()
    good = (a.cpu().numpy().view(np.uint64) == np.atleast_1d(want).view(np.uint64)).all()
    print(f"rank {rank} alpha update: {'match' if good else 'MISMATCH'}", flush=True)
    ok = ok and good
    dist.barrier()
    comm.close()
    dist.destroy_process_group()
    if ok:
        print(f"P2P-OK rank {rank}", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
