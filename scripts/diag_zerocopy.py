"""Diagnostic: the decode step with its inputs in pinned host memory (kernels read them over PCIe,
UVA zero-copy) vs copying all inputs to the device first."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2406_14066_b200.step import SpecStep, StepInputs  # noqa: E402

dev = torch.device("cuda")
B, V, L = 256, 32000, 4096
vb = synth.make_verify_batch(B=B, V=V, k_max=8, lam=0.7, seed=5, device="cpu")
c, o = synth.make_contexts(B=B, L=L, V=V, seed=5)
pin = lambda t: t.contiguous().pin_memory()
hv = synth.VerifyBatch(pin(vb.p), pin(vb.q), pin(vb.row_offsets), pin(vb.draft_tokens), pin(vb.request_ids),
                       vb.k, V, 8)
inp = StepInputs([hv], [pin(torch.tensor(c))], [pin(torch.tensor(o))],
                 [pin(torch.tensor(np.diff(o).astype(np.int32)))], 8)
st = SpecStep(inp, device=dev)
for mode in ("zero-copy",):
    for t in range(3):
        st.run(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for t in range(n):
        st.run(t)
        h = st.num_accepted.cpu()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{mode}: {ms:.3f} ms per step, tokens/step {int((h.numpy() + 1).sum())}, "
          f"{(h.numpy() + 1).sum() / (ms * 1e-3) / 1e3:.0f} k tokens/s")
