"""CPU reference of the closed decode loop (NEXT 4), composed only of oracle/ functions:
lookup -> choose-k (PLD) -> synthetic target (reading R26) -> verify (one-hot drafts) ->
alpha update -> context append.  Used by the GPU closed-loop parity test."""
import numpy as np

import oracle


def run_oracle_loop(ctx0, L, ctx_len0, alpha0, alpha_true, steps, V, K, target, pld_cost_ms, seed,
                    n_min=1, n_max=4, decay=0.9, request_ids=None):
    B = ctx_len0.size
    ctx = np.array(ctx0, np.int32).copy()
    cl = np.array(ctx_len0, np.int32).copy()
    alpha = float(alpha0)
    rid = np.arange(B, dtype=np.uint32) if request_ids is None else np.asarray(request_ids, np.uint32)
    offs = (np.arange(B + 1) * L).astype(np.int32)
    log = []
    for t in range(steps):
        props, plen = oracle.lookup(ctx, offs, n_min, n_max, K)
        kstar, _ = oracle.choose_k(alpha, cl, plen, K, oracle.POLICY_PLD, target, (0.0, 0.0, 0.0),
                                   pld_cost_ms=pld_cost_ms)
        kreq = np.minimum(kstar, plen).astype(np.int32)
        p, ro, d = oracle.sim_target(props, kreq, alpha_true[t], V)
        na, out, st = oracle.verify(p, None, ro, d, rid, seed, t, K)
        alpha = float(oracle.update(alpha, na, ro, decay=decay))
        ctx, cl = oracle.context_append(ctx, L, out, na, cl)
        log.append({"k_star": int(kstar), "num_accepted": na.copy(), "out_tokens": out.copy(), "alpha": alpha,
                    "k_req": kreq.copy(), "proposal_len": plen.copy(), "status": st})
    return log, ctx, cl
