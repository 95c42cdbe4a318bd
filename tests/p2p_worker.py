"""Worker of test_p2p_vocab_shard_two_processes_ipc (launched by torch.distributed.run, 2 ranks).

Both ranks share the box's one GPU; each holds one vocab shard of the same batch, maps the
other's symmetric buffer over CUDA IPC (tsv.P2PComm, handles exchanged over gloo) and runs
tsv_verify_accept_sharded_p2p for several steps; outputs must equal the unsharded oracle."""
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
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
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
    for step in range(4):
        a = tsv.make_verify_args(p, q, g.row_offsets, g.draft_tokens, g.request_ids, 31, step, vb.k_max, na, out,
                                 device_status=st, vocab=Vs, vocab_offset=lo, vocab_global=V)
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
    dist.barrier()
    comm.close()
    dist.destroy_process_group()
    if ok:
        print(f"P2P-OK rank {rank}", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
