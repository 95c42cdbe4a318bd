#!/usr/bin/env python
"""Benchmark of the B200-native TurboSpec decode step (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step = one pass of the whole hot path over one
batch: prompt lookup (256 x 4096-token contexts, n 1-4, K = 5) -> goodput
k-selection (PLD policy) -> rejection-sampling verify/accept (config 2: B = 256,
ragged k in [0, 8], V = 32000, dense fp32 p and q, lambda = 0.7) -> alpha update.
Inputs are seeded synthetic data (synth/), resident in HBM, rotating over R sets
whose footprint is > 3x L2 so no step reads another's rows from L2.
Metric: generated (verified) tokens/s = sum_i (m_i + 1) / time, whole job.
Roofline: the dominant kernel (verify_race_kernel) timed alone -- at least 64 race-only launches per
graph (TSV_VERIFY_RACE_ONLY) over per-step workspaces, at least 4 replays whatever K -- against its
algorithmic bytes (the rows the steps actually select) and MEASURED_PEAKS.json's HBM copy bandwidth;
the whole verify call is reported beside it.  e2e: the same ABI calls with the inputs in pinned host memory.
Timing: W untimed warm-up steps, then exactly K steps (CUDA-graph replays of up to 64 steps) between
CUDA events on the launching stream, bracketed by a barrier + synchronize; a ~50 us spin kernel
enqueued just before the start event keeps the device busy while the host submits the first replay,
so the events time device work only (without it a K = 20 run charged ~1 us per step of graph-launch
latency).
Multi-GPU: one server over the N ranks, request-sharded -- every rank runs B = 256
requests (global request ids) and alpha / k* are GLOBAL: the exact int64 ArgMaxGoodput sums and the
(sum m, sum t) acceptance pair are summed over the ranks through NVLink peer memory inside the
goodput kernel and the verify's update CTA (no NCCL launch; --comm nccl for NCCL all-reduces);
time = max over ranks ("scaling": "weak").  Sub-objects ("workloads"): the strong-scaling line
(one B = 256 batch split by request), config 4 vocab-sharded over the N ranks, greedy, logits,
the config-5 goodput sweep and the closed decode loop, each with its own roofline, clocks and
device status (--no-extras omits them; --workload X prints X alone).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "generated tokens/s (verified, whole job)"
UNIT = "tokens/s"
WORKLOAD = ("config2 verify (B=256, k~U{0..8}, V=32000, fp32 p+q, lambda=0.7) + config3 PLD lookup "
            "(B=256, L=4096, n 1-4, K=5) + goodput choose-k (PLD) + alpha update")
B, V, K_MAX, L_CTX = 256, 32000, 8, 4096


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sets", type=int, default=4, help="rotating input sets (L2 defeat)")
    ap.add_argument("--graph-steps", type=int, default=64, help="decode steps per captured CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--fused", action="store_true", help="fused lookup+choose-k call (verify+update is always one call)")
    ap.add_argument("--no-early-trigger", action="store_true",
                    help="verify without TSV_VERIFY_EARLY_TRIGGER (the next step's lookup launches after the emit)")
    ap.add_argument("--no-lookup-ready", action="store_true",
                    help="launch the lookup without TSV_LOOKUP_INPUTS_READY (its loads wait for the preceding kernel)")
    ap.add_argument("--ld", type=int, default=0,
                    help="row stride (elements) of the step's p / q buffers (default: vocab); layout experiments")
    ap.add_argument("--nvtx", action="store_true",
                    help="NVTX ranges: TSV_NVTX=1 (every libtsv entry point) plus one range per bench phase / workload")
    ap.add_argument("--breakdown", action="store_true", help="also time each step component alone (in graphs)")
    ap.add_argument("--comm", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1 exchange of the request-sharded global sums: NVLink peer memory inside the goodput "
                         "and update kernels (p2p) or NCCL all-reduces (nccl)")
    ap.add_argument("--no-extras", action="store_true",
                    help="omit the other workloads' sub-objects (config4, greedy, logits, config5, loop, strong)")
    ap.add_argument("--workload", default="step",
                    choices=["step", "config4", "greedy", "logits", "config5", "loop", "strong"],
                    help="step: the default decode step; config4: Llama-3 vocab-sharded verify (V=128256) "
                         "through tsv_verify_accept_sharded over the N ranks (strong scaling); greedy: the "
                         "temperature-0 verify (NEXT 2) on the config-2 batch (weak scaling); logits: the fused "
                         "softmax-from-logits verify (NEXT 1) on the config-2 batch given as logits; config5: the "
                         "goodput sweep (B 1-512 x alpha 0.3-0.9, K = 8) as one batched choose-k launch")
    ap.add_argument("--shard-mode", default="auto", choices=["auto", "none", "lazy", "dense", "p2p", "p2p_fused"],
                    help="config4 sharding mode: lazy two rounds over NCCL all-reduces, one-round dense over an "
                         "NCCL all-gather, or the lazy two rounds over NVLink peer memory (no NCCL); none = the "
                         "unsharded tsv_verify_accept (N = 1 only); auto = p2p for N > 1, none for N = 1")
    return ap.parse_args()


# Test mode for the N > 1 host path on a one-GPU box: TSV_BENCH_SHARED_GPU=1 puts every rank on
# cuda:0 and uses the gloo backend (NCCL refuses two ranks on one device).  Not a measurement.
SHARED_GPU = os.environ.get("TSV_BENCH_SHARED_GPU") == "1"


_JSON_OUT = sys.stdout


def _dev_index(local_rank):
    return 0 if SHARED_GPU else local_rank


def _barrier(dist, local_rank):
    if SHARED_GPU:
        dist.barrier()
    else:
        dist.barrier(device_ids=[local_rank])


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------------- algorithmic bytes
def verify_alg_bytes(m, k, dense_q, vocab, k_max):
    """SURVEY.md 8(d) / DESIGN.md 7: bytes the method must move for one verify launch.

    per request: 4V (p row m) + 4V [m < k, dense q] (q row m) + 32 B per tested gather
    (p, and q when dense; tested = m + [m < k]) + metadata 4(k + 3) + outputs 4(k_max + 2)."""
    m = np.asarray(m, np.int64)
    k = np.asarray(k, np.int64)
    rej = (m < k).astype(np.int64)
    tested = m + rej
    per = 4 * vocab * (1 + rej * (1 if dense_q else 0)) + 32 * tested * (2 if dense_q else 1)
    per += 4 * (k + 3) + 4 * (k_max + 2)
    return int(per.sum())


def lookup_alg_bytes(lens, K):
    lens = np.asarray(lens, np.int64)
    return int((4 * lens + 8 + 4 * (K + 1)).sum())


# ------------------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    """Polls NVML SM clocks and throttle reasons from a thread during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def _loop(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.reasons |= int(r) & ~0x1
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.0005)

    def __enter__(self):  # re-entrant: samples of every `with` block accumulate
        if self.ok:
            self._stop.clear()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        names = [n for b, n in self.REASONS.items() if self.reasons & b]
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": int(self.max_mhz), "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------------------- our arm
def prime_stream(stream, cycles=100000):
    """Keep the device busy (a ~50 us spin kernel, outside the timed region) while the host enqueues
    the start event and the first graph replay: the events then time device work only, not the
    host's submission latency of that replay (which a short run -- one replay -- would otherwise
    charge to its K steps)."""
    import torch
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(cycles))


def committed_traffic(workload):
    """DRAM bytes (read + write) per call of a workload's kernels from the committed ncu capture
    (profiles/r02/traffic.json, scripts/traffic.sh: cold caches, per-launch means summed over the call's
    kernels); None when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "traffic.json")) as f:
            return json.load(f)[workload]["dram_bytes_per_call"]
    except Exception:  # noqa: BLE001
        return None


def _sets_for(args, bytes_per_set, l2):
    """Rotating input sets: at least --sets, and enough that R x footprint >= 3 x L2."""
    need = int(np.ceil(3.0 * l2 / max(1, bytes_per_set)))
    return int(min(16, max(args.sets, need)))


def build_step_inputs(mode, rank, world, dev, args, B_total):
    """The step's rotating input sets on this rank.
    weak:   the rank's own B_total requests (global ids rank * B_total + i): one server whose batch
            grows with N (global alpha / k* over all ranks);
    strong: requests [lo, hi) of ONE B_total batch (the same seed on every rank), split by
            dist.partition_requests (balanced sum(2 k_i + 1))."""
    import torch

    import synth
    from paper_2406_14066_b200 import dist as pdist
    from paper_2406_14066_b200.step import StepInputs
    seed = synth.DEFAULT_SEED
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    vbs, ctxs, offs, lens, ks = [], [], [], [], []
    R, s = max(1, args.sets), 0
    while s < R:
        if mode == "weak":
            vb = synth.make_verify_batch(B=B_total, V=V, k_max=K_MAX, lam=0.7, seed=seed + 7919 * s + rank,
                                         device=dev, request_id_base=rank * B_total, ld=args.ld or None)
            c, o = synth.make_contexts(B=B_total, L=L_CTX, V=V, seed=seed + 7919 * s + rank)
            k = vb.k
        else:
            whole = synth.make_verify_batch(B=B_total, V=V, k_max=K_MAX, lam=0.7, seed=seed + 7919 * s, device=dev)
            c, o = synth.make_contexts(B=B_total, L=L_CTX, V=V, seed=seed + 7919 * s)
            lo, hi = pdist.partition_requests(whole.k.cpu().numpy(), world)[rank]
            p, q, ro, d, rid = pdist.request_slice(whole.p, whole.q, whole.row_offsets, whole.draft_tokens,
                                                   whole.request_ids, lo, hi)
            vb = synth.VerifyBatch(p.clone(), q.clone(), ro.clone(), d.clone(), rid.clone(), whole.k[lo:hi].clone(),
                                   V, K_MAX)
            c, o = c[o[lo]:o[hi]], (o[lo:hi + 1] - o[lo]).astype(np.int32)
            k = vb.k
            del whole
        vbs.append(vb)
        ctxs.append(torch.tensor(c, device=dev))
        offs.append(torch.tensor(o, device=dev))
        lens.append(torch.tensor(np.diff(o).astype(np.int32), device=dev))
        ks.append(k.cpu().numpy())
        if s == 0:  # enough sets that R x footprint >= 3 x L2 (strong scaling shrinks the per-rank set)
            R = _sets_for(args, (vb.p.numel() + vb.q.numel()) * 4 + c.size * 4, l2)
        s += 1
    torch.cuda.empty_cache()
    inp = StepInputs(vbs, ctxs, offs, lens, K_MAX, seed=seed)
    return inp, ks, l2


def time_step_graphs(args, st, world, local_rank, dev):
    """Warm-up, then exactly K steps replayed from CUDA graphs (distinct Philox step counters),
    timed with CUDA events on the launching stream between barriers; max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2406_14066_b200 import dist as pdist
    W, K = max(3, args.warmup), args.steps
    gl = max(1, min(args.graph_steps, K))
    st.capture(list(range(0, gl)))  # main graph: steps 0..gl-1 (replayed)
    main_graph = st.graph
    rem = K % gl
    rem_graph = None
    if rem:
        st.capture(list(range(gl, gl + rem)))
        rem_graph = st.graph
    st.reset_state()
    with nvtx_range(args, "warmup"):
        for _ in range((W + gl - 1) // gl):
            main_graph.replay()
        torch.cuda.synchronize()

    def barrier():
        if world > 1:
            _barrier(dist, local_rank)

    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(_dev_index(local_rank))
    barrier()
    torch.cuda.synchronize()
    with sampler, nvtx_range(args, "timed"):
        prime_stream(stream)
        e0.record(stream)
        for _ in range(K // gl):
            main_graph.replay()
        if rem_graph is not None:
            rem_graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    t_max = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
    n_timed_samples = len(sampler.samples)
    # spread: a second pass with an event around every graph replay (kept out of the timed region;
    # 64 replays whatever K, so a short driver run still gets p10/p90), clocks sampled again
    n_rep = 64
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n_rep + 1)]
    barrier()
    with sampler, nvtx_range(args, "spread"):
        prime_stream(stream)
        evs[0].record(stream)
        for r in range(n_rep):
            main_graph.replay()
            evs[r + 1].record(stream)
        torch.cuda.synchronize()
    per_step = sorted(evs[r].elapsed_time(evs[r + 1]) / gl for r in range(n_rep))
    spread = {f"p{q}": per_step[min(n_rep - 1, int(q / 100 * n_rep))] for q in (10, 50, 90)}
    spread["replays"] = n_rep
    spread["steps_per_replay"] = gl
    step_ids = [t for _ in range(K // gl) for t in range(gl)] + [gl + t for t in range(rem)]
    clocks = sampler.summary()
    clocks["samples_timed_region"] = n_timed_samples  # the rest were taken during the spread pass
    return {"t_max": t_max, "W": W, "K": K, "gl": gl, "spread": spread, "step_ids": step_ids,
            "clocks": clocks, "stream": stream}


def step_tokens(st, inp, ks, step_ids, dev, workspace_from=None):
    """Generated tokens and verify algorithmic bytes of exactly the timed steps on this rank (the
    verify outputs do not depend on alpha / k*: a plain verify call per distinct step reproduces them)."""
    import torch

    from paper_2406_14066_b200 import tsv
    R = inp.sets
    per_step_tokens, per_step_vbytes = {}, {}
    Bl = inp.B
    na = torch.empty(Bl, dtype=torch.int32, device=dev)
    outt = torch.empty((Bl, K_MAX + 1), dtype=torch.int32, device=dev)
    for t in sorted(set(step_ids)):
        vb = inp.verify[t % R]
        tsv.tsv_verify_accept(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, inp.seed, t,
                              K_MAX, num_accepted=na, out_tokens=outt, workspace=st.workspace)
        m = na[:inp.B_of(t % R)].cpu().numpy()
        per_step_tokens[t] = int((m + 1).sum())
        per_step_vbytes[t] = verify_alg_bytes(m, ks[t % R], True, V, K_MAX)
    return per_step_tokens, per_step_vbytes


def global_state_consistent(st, world, dev):
    """Every rank must hold the same alpha bits and k* after the timed steps (one server)."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        return True
    mine = torch.tensor([int(st.alpha.view(torch.int64).item()), int(st.k_star.item())], dtype=torch.int64)
    allv = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine.to(dev) if dist.get_backend() == "nccl" else mine)
    return all(bool(torch.equal(a.cpu(), allv[0].cpu())) for a in allv)


def make_comm(args, rank, world, B_max):
    """The request-sharded exchange: NVLink peer memory (default) or NCCL (--comm nccl)."""
    if world <= 1:
        return None
    from paper_2406_14066_b200 import tsv
    if args.comm == "nccl" and not SHARED_GPU:
        return tsv.Comm(rank, world)
    try:
        return tsv.P2PComm(rank, world, B_max=B_max)
    except tsv.TsvError as e:  # every rank raises together (P2PComm agrees on the outcome)
        if SHARED_GPU:
            raise
        print(f"[bench] peer-memory exchange unavailable ({e}); using NCCL", file=sys.stderr)
        return tsv.Comm(rank, world)


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2406_14066_b200 import dist as pdist
    from paper_2406_14066_b200 import tsv
    from paper_2406_14066_b200.step import SpecStep, StepInputs

    import synth
    dev = torch.device("cuda", _dev_index(local_rank))
    torch.cuda.set_device(dev)
    seed = synth.DEFAULT_SEED
    # weak scaling, one server: every rank owns B = 256 requests (global ids), alpha and k* are global
    inp, ks, l2 = build_step_inputs("weak", rank, world, dev, args, B)
    R = inp.sets
    vbs = inp.verify
    comm = make_comm(args, rank, world, B)
    st = SpecStep(inp, device=dev, chunk=args.chunk, fused=args.fused and comm is None, comm=comm,
                  lookup_ready=not args.no_lookup_ready, early_trigger=not args.no_early_trigger)
    footprint = sum(inp.input_bytes(s) for s in range(R))
    tm = time_step_graphs(args, st, world, local_rank, dev)
    t_max, W, K, gl, stream = tm["t_max"], tm["W"], tm["K"], tm["gl"], tm["stream"]
    consistent = global_state_consistent(st, world, dev)

    # ---- generated tokens and algorithmic bytes of exactly the timed steps (deterministic)
    per_step_tokens, per_step_vbytes = step_tokens(st, inp, ks, tm["step_ids"], dev)
    tokens_rank = sum(per_step_tokens[t] for t in tm["step_ids"])
    tokens_total = pdist.sum_over_ranks(tokens_rank, dev)
    value = tokens_total / (t_max / 1e3)
    na = torch.empty(B, dtype=torch.int32, device=dev)
    outt = torch.empty((B, K_MAX + 1), dtype=torch.int32, device=dev)

    # ---- the dominant kernel alone, timed live with CUDA events: graphs of glr >= 64 launches replayed at
    # least 4 times whatever K (a short driver run would otherwise time one replay of a few launches)
    glr = max(gl, 64)
    if glr > gl:  # algorithmic bytes of the extra steps (the step ids the roofline graphs use: 0 .. glr-1)
        _, extra_vbytes = step_tokens(st, inp, ks, [t for t in range(gl, glr)], dev)
        per_step_vbytes = {**per_step_vbytes, **extra_vbytes}
    vgraph = torch.cuda.CUDAGraph()
    ws = st.workspace
    vargs = []
    for t in range(glr):
        s = t % R
        vb = vbs[s]
        a = tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, seed, t,
                                 K_MAX, na, outt, None, ws, chunk=args.chunk, flags=tsv.VERIFY_META_READY)
        vargs.append(a)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        with torch.cuda.graph(vgraph, stream=side):
            for a in vargs:
                tsv._check(tsv.lib().tsv_verify_accept(tsv.ctypes.byref(a), side.cuda_stream))
    torch.cuda.synchronize()
    for _ in range(2):
        vgraph.replay()
    torch.cuda.synchronize()
    reps = max(4, K // glr)
    v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prime_stream(stream)
    v0.record(stream)
    for _ in range(reps):
        vgraph.replay()
    v1.record(stream)
    torch.cuda.synchronize()
    verify_ms = v0.elapsed_time(v1) / (reps * glr)
    vbytes = statistics.fmean(per_step_vbytes[t] for t in range(glr))
    peak, peak_src = load_peaks()
    achieved = vbytes / (verify_ms * 1e-3) / 1e9
    # ---- the race kernel (the dominant kernel of the call) alone: per step t its own workspace holds
    # the scan results of a full call at step t, then gl race-only launches (TSV_VERIFY_RACE_ONLY) in a
    # graph; the race max-combines into the same keys, so it streams exactly the rows of step t again.
    race_ws = [torch.empty_like(ws) for _ in range(glr)]
    rargs = []
    for t in range(glr):
        vb = vbs[t % R]
        a = tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, seed, t,
                                 K_MAX, na, outt, None, race_ws[t], chunk=args.chunk)
        tsv._check(tsv.lib().tsv_verify_accept(tsv.ctypes.byref(a), stream.cuda_stream))
        rargs.append(tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, seed, t,
                                          K_MAX, na, outt, None, race_ws[t], chunk=args.chunk,
                                          flags=tsv.VERIFY_RACE_ONLY))
    torch.cuda.synchronize()
    rgraph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(rgraph, stream=side):
            for a in rargs:
                tsv._check(tsv.lib().tsv_verify_accept(tsv.ctypes.byref(a), side.cuda_stream))
    torch.cuda.synchronize()
    for _ in range(2):
        rgraph.replay()
    torch.cuda.synchronize()
    prime_stream(stream)
    v0.record(stream)
    for _ in range(reps):
        rgraph.replay()
    v1.record(stream)
    torch.cuda.synchronize()
    race_ms = v0.elapsed_time(v1) / (reps * glr)
    race_achieved = vbytes / (race_ms * 1e-3) / 1e9
    del race_ws

    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "verify_traffic.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")  # committed ncu --set full capture
    except Exception:
        pass

    # ---- optional: each step component alone, gl launches per graph (in-graph cost per launch)
    breakdown = None
    if args.breakdown:
        breakdown = {}
        for comp in ("lookup", "choose_k", "verify", "update", "verify_update"):
            if comm is not None and comp in ("update", "verify"):
                continue
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                st.run_component(comp, 0, stream=side)
                torch.cuda.synchronize()
                with torch.cuda.graph(cg, stream=side):
                    for t in range(gl):
                        st.run_component(comp, t, stream=side)
            torch.cuda.synchronize()
            cg.replay()
            torch.cuda.synchronize()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            prime_stream(stream)
            c0.record(stream)
            for _ in range(reps):
                cg.replay()
            c1.record(stream)
            torch.cuda.synchronize()
            breakdown[comp] = round(c0.elapsed_time(c1) / (reps * gl) * 1e3, 3)

    # ---- end to end through the public API with host buffers (pinned): every step reads its inputs from
    # host memory inside the timed region and copies its results back.  Two modes:
    #  zero-copy (reported as "e2e"): the same ABI calls with the inputs left in pinned host memory; the
    #    kernels read exactly the bytes the lazy path needs over PCIe (UVA), counted per step;
    #  full copy ("e2e_full_copy"): cudaMemcpy of every input tensor (all p and q rows) first.
    e2e = e2e_copy = None
    st_h = None
    ctxs, offs, lens = inp.ctx, inp.ctx_offsets, inp.ctx_len
    if args.e2e_steps > 0:
        vb = vbs[0]
        names = ["p", "q", "row_offsets", "draft_tokens", "request_ids"]
        host = [getattr(vb, nm).cpu().pin_memory() for nm in names]
        hctx = [ctxs[0].cpu().pin_memory(), offs[0].cpu().pin_memory(), lens[0].cpu().pin_memory()]
        out_host = [torch.empty((B, K_MAX + 1), dtype=torch.int32).pin_memory(),
                    torch.empty(B, dtype=torch.int32).pin_memory(),
                    torch.empty(1, dtype=torch.float64).pin_memory()]
        d2h = sum(t.numel() * t.element_size() for t in out_host)
        ne = args.e2e_steps
        hv = synth.VerifyBatch(host[0], host[1], host[2], host[3], host[4], vb.k, V, K_MAX)
        st_h = SpecStep(StepInputs([hv], [hctx[0]], [hctx[1]], [hctx[2]], K_MAX, seed=seed), device=dev,
                        chunk=args.chunk, comm=comm, lookup_ready=not args.no_lookup_ready,
                        early_trigger=not args.no_early_trigger)
        k_np = ks[0]
        ctx_bytes = hctx[0].numel() * 4 + hctx[1].numel() * 4 + hctx[2].numel() * 4

        def run_e2e(step_fn, outs_from):
            toks, h2d_zc = 0, 0
            torch.cuda.synchronize()
            if world > 1:
                import torch.distributed as dist
                _barrier(dist, local_rank)
            w0 = time.perf_counter()
            x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x0.record(stream)
            for t in range(ne):
                step_fn(t)
                out_host[0].copy_(outs_from.out_tokens, non_blocking=True)
                out_host[1].copy_(outs_from.num_accepted, non_blocking=True)
                out_host[2].copy_(outs_from.alpha, non_blocking=True)
                stream.synchronize()
                m = out_host[1].numpy()
                toks += int((m + 1).sum())
                h2d_zc += verify_alg_bytes(m, k_np, True, V, K_MAX) + ctx_bytes
            x1.record(stream)
            torch.cuda.synchronize()
            e_ms = pdist.max_over_ranks(x0.elapsed_time(x1), dev)
            return pdist.sum_over_ranks(toks, dev) / (e_ms / 1e3), h2d_zc / ne, time.perf_counter() - w0

        val, h2d_zc, wall = run_e2e(lambda t: st_h.run(step=t), st_h)
        e2e = {"value": val, "unit": UNIT, "h2d_bytes_per_step": int(h2d_zc), "d2h_bytes_per_step": int(d2h),
               "steps": ne, "wall_s": round(wall, 4),
               "mode": "zero-copy: inputs stay in pinned host memory; the kernels read the lazy path's bytes "
                       "over PCIe (UVA), outputs copied back"}

        def full_copy_step(t):
            for nm, h in zip(names, host):
                getattr(vb, nm).copy_(h, non_blocking=True)
            ctxs[0].copy_(hctx[0], non_blocking=True)
            offs[0].copy_(hctx[1], non_blocking=True)
            lens[0].copy_(hctx[2], non_blocking=True)
            st.run(step=t * R)  # set 0

        val_c, _, wall_c = run_e2e(full_copy_step, st)
        e2e_copy = {"value": val_c, "unit": UNIT,
                    "h2d_bytes_per_step": int(sum(t.numel() * t.element_size() for t in host + hctx)),
                    "d2h_bytes_per_step": int(d2h), "steps": ne, "wall_s": round(wall_c, 4),
                    "mode": "cudaMemcpy of every input tensor (all p and q rows) each step"}
    st_status = int(pdist.max_over_ranks(int(st.status.item()), dev))
    del st, st_h
    close_comm(comm, world, local_rank)
    if rank != 0:
        return None
    par = "request-sharded x1" if world == 1 else (
        f"request-sharded x{world}, one server: global alpha / k* through "
        + ("NVLink peer memory inside the goodput and update kernels (p2p)" if comm is not None and
           not isinstance(comm, tsv.Comm) else "NCCL all-reduce (nccl)"))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": t_max / K, "ms_per_step_spread": tm["spread"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, synth/)",
        "config": {"workload": WORKLOAD, "global_batch": B * world, "vocab": V, "k_max": K_MAX,
                   "ctx_len": L_CTX, "parallelism": par,
                   "l2_defeat": f"{R} rotating input sets, footprint {footprint / 1e6:.0f} MB vs L2 {l2 / 1e6:.0f} MB",
                   "graph_steps": gl, "fused": bool(args.fused and comm is None),
                   "lookup_inputs_ready": not args.no_lookup_ready,
                   "verify_early_trigger": not (args.no_early_trigger or args.no_lookup_ready)},
        "roofline": {"kernel": "verify_race_kernel (the dominant kernel: streams every algorithmic byte of the verify call)",
                     "bound": "hbm", "achieved": race_achieved, "peak": peak,
                     "unit": "GB/s", "frac": race_achieved / peak, "traffic": traffic,
                     "alg_bytes_per_launch": vbytes, "launch_us": race_ms * 1e3, "peak_source": peak_src,
                     "verify_call": {"kernels": "verify_scan + verify_race + verify_emit", "launch_us": verify_ms * 1e3,
                                     "achieved": achieved, "frac": achieved / peak}},
        "clocks": tm["clocks"],
        "gpu_launches": st_launches(comm, args) * K,
        "e2e": e2e,
        "e2e_full_copy": e2e_copy,
        "tokens_per_step": tokens_total / K,
        "requests_per_s": B * world * K / (t_max / 1e3),
        "device_status": st_status,
        "global_state_consistent": consistent,
    }
    if breakdown is not None:
        line["breakdown_us_per_launch"] = breakdown
    return line


def close_comm(comm, world, local_rank):
    """Every rank's exchanges are complete (streams synchronised) before any buffer is freed."""
    if comm is None:
        return
    import torch
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        _barrier(dist, local_rank)
    comm.close()


def st_launches(comm, args):
    from paper_2406_14066_b200 import tsv
    if comm is not None and isinstance(comm, tsv.Comm):
        return 10
    return 4 if (args.fused and comm is None) else 5


def run_strong(args, rank, world, local_rank):
    """Strong scaling: ONE B = 256 batch split across the N ranks by request
    (partition_requests), global alpha / k* through the same exchange as the weak line."""
    import torch

    from paper_2406_14066_b200 import dist as pdist
    from paper_2406_14066_b200.step import SpecStep
    dev = torch.device("cuda", _dev_index(local_rank))
    torch.cuda.set_device(dev)
    inp, ks, l2 = build_step_inputs("strong", rank, world, dev, args, B)
    comm = make_comm(args, rank, world, B)
    st = SpecStep(inp, device=dev, chunk=args.chunk, comm=comm, lookup_ready=not args.no_lookup_ready,
                  early_trigger=not args.no_early_trigger)
    tm = time_step_graphs(args, st, world, local_rank, dev)
    consistent = global_state_consistent(st, world, dev)
    per_step_tokens, per_step_vbytes = step_tokens(st, inp, ks, tm["step_ids"], dev)
    tokens_total = pdist.sum_over_ranks(sum(per_step_tokens[t] for t in tm["step_ids"]), dev)
    vbytes = pdist.sum_over_ranks(sum(per_step_vbytes[t] for t in tm["step_ids"]), dev) / tm["K"]
    lbytes = pdist.sum_over_ranks(lookup_alg_bytes(inp.ctx_len[0].cpu().numpy(), inp.k_fixed), dev)
    st_status = int(pdist.max_over_ranks(int(st.status.item()), dev))
    footprint = sum(inp.input_bytes(s) for s in range(inp.sets))
    R, Bl = inp.sets, inp.B
    del st
    close_comm(comm, world, local_rank)
    if rank != 0:
        return None
    t_max, K = tm["t_max"], tm["K"]
    ms = t_max / K
    peak, peak_src = load_peaks()
    step_bytes = vbytes + lbytes
    achieved = step_bytes / (ms * 1e-3) / 1e9
    return {
        "metric": METRIC, "value": tokens_total / (t_max / 1e3), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": tm["W"], "ms_per_step": ms, "ms_per_step_spread": tm["spread"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, synth/)",
        "config": {"workload": WORKLOAD + f" -- one B={B} batch split by request over {world} ranks",
                   "global_batch": B, "local_batch_rank0": Bl, "vocab": V, "k_max": K_MAX, "ctx_len": L_CTX,
                   "parallelism": f"request-sharded x{world} (strong), global alpha / k* over the ranks",
                   "l2_defeat": f"{R} rotating input sets, rank 0 footprint {footprint / 1e6:.0f} MB vs L2 {l2 / 1e6:.0f} MB",
                   "graph_steps": tm["gl"]},
        "roofline": {"kernel": "whole step per rank (lookup + choose-k + verify + update)", "bound": "hbm",
                     "achieved": achieved, "peak": peak * world, "unit": "GB/s", "frac": achieved / (peak * world),
                     "traffic": None, "alg_bytes_per_launch": step_bytes, "launch_us": ms * 1e3,
                     "peak_source": peak_src + f" x {world} GPUs"},
        "clocks": tm["clocks"], "gpu_launches": st_launches(comm, args) * K, "e2e": None,
        "tokens_per_step": tokens_total / K, "requests_per_s": B * K / (t_max / 1e3), "device_status": st_status,
        "global_state_consistent": consistent,
    }


# ------------------------------------------------------------------ config 4 (vocab sharded)
V4 = 128256


def run_config4(args, rank, world, local_rank):
    """BASELINE config 4: one B = 256 batch at V = 128256, vocab-sharded over the N ranks as under a
    tensor-parallel LM head (rank g holds columns [g V/N, (g+1) V/N) of every p/q row); one step =
    tsv_verify_accept_sharded (lazy: flags -> NCCL all-reduce(sum) -> race of row m -> NCCL
    all-reduce(max) -> emit; dense: partial -> NCCL all-gather -> combine).  Strong scaling."""
    import torch

    import synth
    from paper_2406_14066_b200 import dist as pdist
    from paper_2406_14066_b200 import tsv

    dev = torch.device("cuda", _dev_index(local_rank))
    torch.cuda.set_device(dev)
    R = max(2, args.sets)
    seed = synth.DEFAULT_SEED
    lo, Vs = pdist.vocab_shards(V4, world)[rank]
    hi = lo + Vs
    if args.shard_mode == "auto":
        args.shard_mode = "p2p" if world > 1 else "none"
    if args.shard_mode == "none" and world > 1:
        raise SystemExit("--shard-mode none is the one-GPU (unsharded) call")
    p2p = args.shard_mode in ("p2p", "p2p_fused")
    unsharded = args.shard_mode == "none"
    comm = None
    if not unsharded and p2p:
        try:
            comm = tsv.P2PComm(rank, world, B_max=B)
        except tsv.TsvError as e:  # every rank raises together: fall back to the NCCL lazy mode
            if SHARED_GPU:
                raise
            print(f"[bench] peer-memory exchange unavailable ({e}); config 4 uses the NCCL lazy mode", file=sys.stderr)
            p2p = False
            args.shard_mode = "lazy"
    if not unsharded and not p2p:
        comm = tsv.Comm(rank, world)
    flags = tsv.VERIFY_SHARD_DENSE if args.shard_mode == "dense" else 0
    if args.shard_mode == "p2p_fused":  # the race items push their chunk keys (no keys kernel)
        flags = tsv.VERIFY_P2P_FUSED
    if unsharded:  # the batch's offsets / drafts / ids are inputs, not written by the preceding kernel
        flags = tsv.VERIFY_META_READY
    entry = tsv.lib().tsv_verify_accept_sharded_p2p if p2p else tsv.lib().tsv_verify_accept_sharded

    def run_sharded(a, stream=None):
        if unsharded:  # one GPU holds the whole vocabulary: scan -> race -> emit, no exchange
            tsv._check(tsv.lib().tsv_verify_accept(tsv.ctypes.byref(a), tsv._stream(stream)))
        else:
            tsv._check(entry(tsv.ctypes.byref(a), comm.handle, tsv._stream(stream)))
    na = torch.empty(B, dtype=torch.int32, device=dev)
    outt = torch.empty((B, K_MAX + 1), dtype=torch.int32, device=dev)
    dstat = torch.zeros(1, dtype=torch.int32, device=dev)
    sets, footprint = [], 0
    for s in range(R):  # the same logical batch on every rank (same seed), this rank's columns kept
        vb = synth.make_verify_batch(B=B, V=V4, k_max=K_MAX, lam=0.7, seed=seed + 104729 * s, device=dev)
        p = vb.p[:, lo:hi].contiguous()
        q = vb.q[:, lo:hi].contiguous()
        footprint += (p.numel() + q.numel()) * 4
        sets.append((vb, p, q))
        del vb.p, vb.q
    torch.cuda.empty_cache()
    args_list = []
    W, K = max(3, args.warmup), args.steps
    gl = max(1, min(args.graph_steps, K))
    for t in range(gl):
        vb, p, q = sets[t % R]
        a = tsv.make_verify_args(p, q, vb.row_offsets, vb.draft_tokens, vb.request_ids, seed, t, K_MAX, na, outt,
                                 dstat, None, vocab=Vs, vocab_offset=lo, vocab_global=V4, chunk=args.chunk,
                                 flags=flags)
        args_list.append(a)
    ws = tsv.alloc_workspace(max(tsv.tsv_verify_sharded_workspace_size(a, world) for a in args_list), dev)
    for a in args_list:
        a.workspace = ws.data_ptr()
        a.workspace_bytes = ws.numel()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        run_sharded(args_list[0], stream=side)  # warm-up outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for a in args_list:
            run_sharded(a, stream=side)
    torch.cuda.synchronize()
    for _ in range((W + gl - 1) // gl):
        g.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, K // gl)
    sampler = ClockSampler(local_rank)
    def barrier():
        if world > 1:
            import torch.distributed as dist
            _barrier(dist, local_rank)

    barrier()
    torch.cuda.synchronize()
    with sampler:
        prime_stream(stream)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    t_ms = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
    steps = reps * gl
    # tokens and algorithmic bytes of the timed steps (identical on every rank)
    tok, vbytes = 0, 0.0
    for t in range(gl):
        a = args_list[t]
        run_sharded(a)
        torch.cuda.synchronize()
        m = na.cpu().numpy()
        k = sets[t % R][0].k.cpu().numpy()
        tok += int((m + 1).sum())
        dense = args.shard_mode == "dense"
        rows = (2 * k + 1) if dense else (1 + (m < k))  # rows streamed per request (all ranks together)
        vbytes += float((rows * V4 * 4).sum()) / world
    tok_per_step, vbytes = tok / gl, vbytes / gl
    ms_step = t_ms / steps
    st_status = int(pdist.max_over_ranks(int(dstat.item()), dev))
    del sets
    close_comm(comm, world, local_rank)
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    peak, peak_src = load_peaks()
    achieved = vbytes / (ms_step * 1e-3) / 1e9
    return {
        "metric": METRIC, "value": tok_per_step / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": W, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, synth/)",
        "config": {"workload": f"config4 Llama-3 verify (B={B}, k~U{{0..{K_MAX}}}, V={V4}, fp32 p+q, lambda=0.7), "
                               + ("one GPU, unsharded" if unsharded else f"vocab-sharded x{world} ({args.shard_mode})"),
                   "global_batch": B, "vocab": V4, "k_max": K_MAX,
                   "parallelism": "unsharded x1" if unsharded else f"vocab-sharded x{world} ({args.shard_mode})",
                   "l2_defeat": f"{R} rotating input sets, {footprint / 1e6:.0f} MB per rank",
                   "graph_steps": gl},
        "roofline": {"kernel": "tsv_verify_accept (unsharded, one GPU)" if unsharded else
                     f"tsv_verify_accept_sharded{'_p2p' if p2p else ''} (per rank)", "bound": "hbm",
                     "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": committed_traffic("config4") if unsharded else None,
                     "alg_bytes_per_launch": vbytes, "launch_us": ms_step * 1e3, "peak_source": peak_src},
        "clocks": sampler.summary(),
        "gpu_launches": (3 if (args.shard_mode == "dense" or unsharded) else 5) * steps,
        "e2e": None,
        "tokens_per_step": tok_per_step,
        "requests_per_s": B / (ms_step * 1e-3),
        "device_status": st_status,
    }


# ------------------------------------------------------------------ greedy verify (NEXT 2)
def run_greedy(args, rank, world, local_rank):
    """tsv_verify_greedy on the config-2 batch (B = 256, k ~ U{0..8}, V = 32000, fp32 p; drafts
    equal the target argmax w.p. 0.7).  Every p row is streamed (each needs its argmax)."""
    import torch

    import synth
    from paper_2406_14066_b200 import dist as pdist
    from paper_2406_14066_b200 import tsv

    dev = torch.device("cuda", _dev_index(local_rank))
    torch.cuda.set_device(dev)
    R = max(2, args.sets)
    sets, footprint = [], 0
    for s in range(R):
        vb = synth.make_verify_batch(B=B, V=V, k_max=K_MAX, lam=0.7, seed=synth.DEFAULT_SEED + 31 * s + rank,
                                     device=dev, request_id_base=rank * B)
        am = vb.p.argmax(dim=1).to(torch.int32)
        ro = vb.row_offsets.long()
        g = torch.Generator(device="cpu").manual_seed(1000 + s + 7 * rank)
        keep = torch.rand(vb.draft_tokens.numel(), generator=g) < 0.7
        rows = torch.cat([torch.arange(int(ro[i]), int(ro[i + 1]) - 1) for i in range(B)]).to(dev)
        d = torch.where(keep.to(dev), am[rows], vb.draft_tokens)
        footprint += vb.p.numel() * 4
        sets.append((vb.p, vb.row_offsets, d.contiguous(), vb.k))
        del vb.q
    torch.cuda.empty_cache()
    na = torch.empty(B, dtype=torch.int32, device=dev)
    outt = torch.empty((B, K_MAX + 1), dtype=torch.int32, device=dev)
    dstat = torch.zeros(1, dtype=torch.int32, device=dev)
    W, K = max(3, args.warmup), args.steps
    gl = max(1, min(args.graph_steps, K))
    args_list = []
    for t in range(gl):
        p, ro, d, _ = sets[t % R]
        rids = torch.zeros(B, dtype=torch.int32, device=dev)
        args_list.append(tsv.make_verify_args(p, None, ro, d, rids, 0, 0, K_MAX, na, outt, dstat, None,
                                              chunk=args.chunk))
    ws = tsv.alloc_workspace(max(tsv.tsv_verify_workspace_size(a) for a in args_list), dev)
    for a in args_list:
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        tsv._check(tsv.lib().tsv_verify_greedy(tsv.ctypes.byref(args_list[0]), side.cuda_stream))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for a in args_list:
            tsv._check(tsv.lib().tsv_verify_greedy(tsv.ctypes.byref(a), side.cuda_stream))
    for _ in range((W + gl - 1) // gl):
        g.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, K // gl)
    sampler = ClockSampler(local_rank)
    if world > 1:
        import torch.distributed as dist
        _barrier(dist, local_rank)
    torch.cuda.synchronize()
    with sampler:
        prime_stream(stream)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    t_ms = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
    steps = reps * gl
    tok, vbytes = 0, 0.0
    for t in range(gl):
        tsv._check(tsv.lib().tsv_verify_greedy(tsv.ctypes.byref(args_list[t]), None))
        torch.cuda.synchronize()
        k = sets[t % R][3].cpu().numpy()
        tok += int((na.cpu().numpy() + 1).sum())
        vbytes += float(((k + 1) * V * 4).sum() + 4 * (k.sum() + 2 * B + 1) + 4 * B * (K_MAX + 2))
    tok_total = pdist.sum_over_ranks(tok, dev) / gl
    vbytes /= gl
    ms_step = t_ms / steps
    st_status = int(pdist.max_over_ranks(int(dstat.item()), dev))
    del sets
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    peak, peak_src = load_peaks()
    achieved = vbytes / (ms_step * 1e-3) / 1e9
    return {
        "metric": METRIC, "value": tok_total / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": W, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, synth/)", "device_status": st_status,
        "config": {"workload": f"greedy verify (temperature 0, NEXT 2): B={B}, k~U{{0..{K_MAX}}}, V={V}, fp32 p, "
                               f"drafts = target argmax w.p. 0.7", "global_batch": B * world, "vocab": V,
                   "k_max": K_MAX, "parallelism": f"request-sharded x{world}",
                   "l2_defeat": f"{R} rotating input sets, {footprint / 1e6:.0f} MB per rank", "graph_steps": gl},
        "roofline": {"kernel": "tsv_verify_greedy (argmax + emit)", "bound": "hbm", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": committed_traffic("greedy"),
                     "alg_bytes_per_launch": vbytes, "launch_us": ms_step * 1e3, "peak_source": peak_src},
        "clocks": sampler.summary(),
        "gpu_launches": 2 * steps,
        "e2e": None,
        "tokens_per_step": tok_total,
        "requests_per_s": B * world / (ms_step * 1e-3),
    }


# ------------------------------------------------------------ fused softmax from logits (NEXT 1)
def run_logits(args, rank, world, local_rank):
    """tsv_verify_accept_logits on the config-2 batch with p and q given as logits (temperature 1):
    one dense statistics pass over every p and q row, then the lazy race of row m from logits."""
    import torch

    import synth
    from paper_2406_14066_b200 import dist as pdist
    from paper_2406_14066_b200 import tsv

    dev = torch.device("cuda", _dev_index(local_rank))
    torch.cuda.set_device(dev)
    R = max(2, args.sets)
    seed = synth.DEFAULT_SEED
    sets, footprint = [], 0
    for s in range(R):
        vb = synth.make_logits_batch(B=B, V=V, k_max=K_MAX, lam=0.7, seed=seed + 53 * s + rank, device=dev)
        vb.request_ids += rank * B
        footprint += (vb.p.numel() + vb.q.numel()) * 4
        sets.append(vb)
    na = torch.empty(B, dtype=torch.int32, device=dev)
    outt = torch.empty((B, K_MAX + 1), dtype=torch.int32, device=dev)
    dstat = torch.zeros(1, dtype=torch.int32, device=dev)
    W, K = max(3, args.warmup), args.steps
    gl = max(1, min(args.graph_steps, K))
    args_list = []
    for t in range(gl):
        vb = sets[t % R]
        args_list.append(tsv.make_verify_args(vb.p, vb.q, vb.row_offsets, vb.draft_tokens, vb.request_ids, seed, t,
                                              K_MAX, na, outt, dstat, None, chunk=args.chunk))
    ws = tsv.alloc_workspace(max(tsv.tsv_verify_logits_workspace_size(a) for a in args_list), dev)
    for a in args_list:
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    L = tsv.lib()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        tsv._check(L.tsv_verify_accept_logits(tsv.ctypes.byref(args_list[0]), 1.0, side.cuda_stream))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for a in args_list:
            tsv._check(L.tsv_verify_accept_logits(tsv.ctypes.byref(a), 1.0, side.cuda_stream))
    for _ in range((W + gl - 1) // gl):
        g.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, K // gl)
    sampler = ClockSampler(local_rank)
    if world > 1:
        import torch.distributed as dist
        _barrier(dist, local_rank)
    torch.cuda.synchronize()
    with sampler:
        prime_stream(stream)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    t_ms = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
    steps = reps * gl
    tok, vbytes = 0, 0.0
    for t in range(gl):
        tsv._check(L.tsv_verify_accept_logits(tsv.ctypes.byref(args_list[t]), 1.0, None))
        torch.cuda.synchronize()
        vb = sets[t % R]
        m = na.cpu().numpy()
        k = vb.k.cpu().numpy()
        tok += int((m + 1).sum())
        # every p and q row once (statistics) + row m of p (and q on a rejection) again (the race)
        vbytes += float(((2 * k + 1) * V * 4).sum() + verify_alg_bytes(m, k, True, V, K_MAX))
    tok_total = pdist.sum_over_ranks(tok, dev) / gl
    vbytes /= gl
    ms_step = t_ms / steps
    st_status = int(pdist.max_over_ranks(int(dstat.item()), dev))
    del sets
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    peak, peak_src = load_peaks()
    achieved = vbytes / (ms_step * 1e-3) / 1e9
    return {
        "metric": METRIC, "value": tok_total / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": W, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, synth/)", "device_status": st_status,
        "config": {"workload": f"fused softmax-from-logits verify (NEXT 1): B={B}, k~U{{0..{K_MAX}}}, V={V}, "
                               f"fp32 target and draft logits, temperature 1, lambda=0.7",
                   "global_batch": B * world, "vocab": V, "k_max": K_MAX, "parallelism": f"request-sharded x{world}",
                   "l2_defeat": f"{R} rotating input sets, {footprint / 1e6:.0f} MB per rank", "graph_steps": gl},
        "roofline": {"kernel": "tsv_verify_accept_logits (stats + scan + race + emit)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": committed_traffic("logits"),
                     "alg_bytes_per_launch": vbytes, "launch_us": ms_step * 1e3, "peak_source": peak_src},
        "clocks": sampler.summary(),
        "gpu_launches": 4 * steps,
        "e2e": None,
        "tokens_per_step": tok_total,
        "requests_per_s": B * world / (ms_step * 1e-3),
    }


# ------------------------------------------------------------------ config 5 (goodput sweep)
def run_config5(args, rank, world, local_rank):
    """BASELINE config 5: ArgMaxGoodput over batch sizes 1-512 x alpha {0.3..0.9} with K = 8 (SPEC desk
    profiles, draft policy, ctx_len ~ U[128, 4096]) -- 3584 independent instances, 919 296 requests --
    as one tsv_goodput_choose_k_batched launch per step.  Instances are split across ranks (weak)."""
    import torch

    import synth
    from paper_2406_14066_b200 import dist as pdist
    from paper_2406_14066_b200 import tsv

    dev = torch.device("cuda", _dev_index(local_rank))
    torch.cuda.set_device(dev)
    alphas = (0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9)
    ctxs, caps, offs, al = [], [], [0], []
    for Bi in range(1, 513):
        ctx, cap = synth.make_goodput_instance(Bi, 8, seed=Bi + 7 * rank)
        for a in alphas:
            ctxs.append(ctx)
            caps.append(cap)
            offs.append(offs[-1] + Bi)
            al.append(a)
    n_inst, n_req = len(al), offs[-1]
    A = torch.tensor(al, dtype=torch.float64, device=dev)
    C = torch.tensor(np.concatenate(ctxs), device=dev)
    P = torch.tensor(np.concatenate(caps), device=dev)
    O = torch.tensor(np.array(offs, np.int32), device=dev)
    k_out = torch.empty(n_inst, dtype=torch.int32, device=dev)
    g_out = torch.empty((n_inst, 9), dtype=torch.float64, device=dev)
    L = tsv.lib()
    tgt, drf = tsv.LatencyModel(*synth.SPEC_DESK_TARGET), tsv.LatencyModel(*synth.SPEC_DESK_DRAFT)

    def launch(st):
        tsv._check(L.tsv_goodput_choose_k_batched(A.data_ptr(), C.data_ptr(), P.data_ptr(), O.data_ptr(), n_inst, 8,
                                                  tsv.POLICY_DRAFT, tgt, drf, 0.0, -1, k_out.data_ptr(),
                                                  g_out.data_ptr(), None, st))

    W, K = max(3, args.warmup), args.steps
    gl = max(1, min(args.graph_steps, K))
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        launch(side.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(gl):
            launch(side.cuda_stream)
    for _ in range((W + gl - 1) // gl):
        g.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, K // gl)
    sampler = ClockSampler(local_rank)
    if world > 1:
        import torch.distributed as dist
        _barrier(dist, local_rank)
    torch.cuda.synchronize()
    with sampler:
        prime_stream(stream)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    t_ms = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
    steps = reps * gl
    ms_step = t_ms / steps
    inst_total = pdist.sum_over_ranks(n_inst, dev)
    if rank != 0:
        return None
    bytes_step = n_req * 8 + n_inst * (8 + 4 + 4 + 9 * 8)  # ctx_len + cap per request; alpha, offsets, outputs
    peak, peak_src = load_peaks()
    achieved = bytes_step / (ms_step * 1e-3) / 1e9
    return {
        "metric": "goodput selections/s (instances, whole job)", "value": inst_total / (ms_step * 1e-3),
        "unit": "instances/s", "n_gpus": world, "steps": steps, "warmup": W, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth/)",
        "config": {"workload": f"config5 goodput sweep: B 1-512 x alpha 0.3-0.9 x K=8, draft policy, SPEC desk profiles "
                               f"({n_inst} instances, {n_req} requests per rank, one batched launch)",
                   "parallelism": f"instance-sharded x{world}", "graph_steps": gl,
                   "l2_defeat": "none: latency/ALU-bound, 7.4 MB of inputs stay L2-resident (stated, not hidden)"},
        "roofline": {"kernel": "goodput_choose_k_batched_kernel", "bound": "latency", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": committed_traffic("config5"),
                     "alg_bytes_per_launch": bytes_step, "launch_us": ms_step * 1e3, "peak_source": peak_src,
                     "note": "one CTA per instance (3 waves of 8 CTAs/SM), each a dependent chain: loads, fp64 "
                             "Horner, int64 reductions, argmax, stores; the HBM fraction is reported, not targeted"},
        "clocks": sampler.summary(),
        "gpu_launches": steps,
        "e2e": None,
        "requests_per_s": n_req * world / (ms_step * 1e-3),
        "device_status": None,
        "device_status_note": "tsv_goodput_choose_k_batched has no device-side data-error path (inputs are counts)",
    }


# ------------------------------------------------------------- closed decode loop (NEXT 4)
def run_loop(args, rank, world, local_rank):
    """The closed loop (paper_2406_14066_b200/loop.py) timed per step: lookup ->
    choose-k (PLD, cap = proposal lengths, alpha of the previous step) -> tsv_sim_target (the synthetic
    target's rows: the stand-in for the model forward, each draft kept w.p. alpha_true = 0.7) -> verify +
    alpha update -> context append; B = 256 contexts of 4096 tokens, V = 32000, K = 5.  T = 64 steps per
    CUDA graph, the graph starting from the initial state so every replay repeats the same 64 steps
    (the generated tokens of a logged replay are exactly those of every timed replay).  Weak scaling."""
    import torch

    import synth
    from paper_2406_14066_b200 import dist as pdist
    from paper_2406_14066_b200.loop import ClosedLoop

    dev = torch.device("cuda", _dev_index(local_rank))
    torch.cuda.set_device(dev)
    T, K, Lc = 64, 5, L_CTX
    ctx, _ = synth.make_contexts(B=B, L=Lc, V=V, seed=synth.DEFAULT_SEED + 17 * rank)
    lp = ClosedLoop(ctx, Lc, np.full(B, Lc, np.int32), V, K, synth.SPEC_DESK_TARGET, 0.05, [0.7] * T, alpha0=0.7,
                    seed=synth.DEFAULT_SEED + rank, device=dev)
    lp.capture(log=True, with_reset=True)  # logged replay: tokens, k*, bytes
    lp.graph.replay()
    torch.cuda.synchronize()
    logs = lp.logs()
    lp.capture(log=False, with_reset=True)
    W, Kst = max(3, args.warmup), args.steps
    reps = max(1, (Kst + T - 1) // T)
    for _ in range(max(1, (W + T - 1) // T)):
        lp.graph.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(_dev_index(local_rank))
    if world > 1:
        import torch.distributed as dist
        _barrier(dist, local_rank)
    torch.cuda.synchronize()
    with sampler:
        prime_stream(stream)
        e0.record(stream)
        for _ in range(reps):
            lp.graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    steps = reps * T
    t_ms = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
    m, kreq = logs["num_accepted"], logs["k_req"]
    tok = int((m + 1).sum())  # per replay (T steps)
    # algorithmic bytes per step: lookup (contexts) + the synthetic target rows actually used (written)
    # + the lazy verify with one-hot drafts (row m of p; one gather per tested position) + the context
    # append (read + write of every window)
    rows = (kreq + 1).sum(axis=1)
    vb = [verify_alg_bytes(m[t], kreq[t], False, V, K) for t in range(T)]
    per_step = [lookup_alg_bytes(np.full(B, Lc), K) + int(rows[t]) * V * 4 + vb[t] + 2 * 4 * Lc * B for t in range(T)]
    st_status = int(pdist.max_over_ranks(int(lp.status.item()), dev))
    tok_total = pdist.sum_over_ranks(tok, dev) * reps
    if rank != 0:
        return None
    ms = t_ms / steps
    peak, peak_src = load_peaks()
    alg = float(np.mean(per_step))
    achieved = alg / (ms * 1e-3) / 1e9
    return {
        "metric": METRIC, "value": tok_total / (t_ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded, synth/; synthetic target rows from tsv_sim_target)",
        "config": {"workload": f"closed decode loop (NEXT 4): B={B} x {Lc}-token contexts, V={V}, K={K} PLD, "
                               f"alpha_true=0.7, {T} steps per graph", "global_batch": B * world, "vocab": V,
                   "parallelism": f"independent loops x{world}", "graph_steps": T,
                   "l2_defeat": "none needed: every step writes 197 MB of synthetic target rows (> L2)"},
        "roofline": {"kernel": "whole closed-loop step (lookup, choose-k, sim_target, verify + update, append)",
                     "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "alg_bytes_per_launch": alg, "launch_us": ms * 1e3, "peak_source": peak_src,
                     "note": "tsv_sim_target writes all B (K+1) rows (197 MB); only the used rows count as algorithmic"},
        "clocks": sampler.summary(), "gpu_launches": 8 * steps, "e2e": None,
        "tokens_per_step": tok / T, "k_star_mean": float(np.mean(logs["k_star"])),
        "alpha_last": float(logs["alpha"][-1]), "device_status": st_status,
    }


# ------------------------------------------------------------------------- oracle (CPU)
def oracle_step_sample(n_req, seed, step, data):
    """One bounded oracle step over the first n_req requests of the workload (CPU)."""
    import oracle
    import synth
    vb, ctx, offs = data
    ro = vb.row_offsets.numpy()
    r_hi = int(ro[n_req])
    q_hi = r_hi - n_req
    c_hi = int(offs[n_req])
    props, plen = oracle.lookup(ctx[:c_hi], offs[:n_req + 1], 1, 4, 5)
    ctx_len = np.diff(offs[:n_req + 1]).astype(np.int32)
    k, _ = oracle.choose_k(0.7, ctx_len, plen, 5, oracle.POLICY_PLD, synth.SPEC_DESK_TARGET,
                           synth.SPEC_DESK_DRAFT, pld_cost_ms=0.05)
    na, out, _ = oracle.verify(vb.p[:r_hi].numpy(), vb.q[:q_hi].numpy(), ro[:n_req + 1],
                               vb.draft_tokens[:q_hi].numpy(), vb.request_ids[:n_req].numpy().view(np.uint32),
                               seed, step, K_MAX)
    oracle.update(0.7, na, ro[:n_req + 1])
    return int((na + 1).sum())


def cpu_data():
    import synth
    vb = synth.make_verify_batch(B=B, V=V, k_max=K_MAX, lam=0.7, seed=synth.DEFAULT_SEED, device="cpu")
    ctx, offs = synth.make_contexts(B=B, L=L_CTX, V=V, seed=synth.DEFAULT_SEED)
    return vb, ctx, offs


def oracle_step_threaded(seed, step, data, pool, T, n_req=B):
    """One oracle step of the bench workload (its first n_req requests) on T host threads: the
    requests are independent (Philox keyed by request id), so contiguous request ranges run the
    oracle's lookup and verify concurrently (ctypes releases the GIL); choose-k and the alpha
    update take all n_req requests."""
    import oracle
    import synth
    vb, ctx, offs = data
    ro = vb.row_offsets.numpy()[:n_req + 1]
    offs = offs[:n_req + 1]
    p, q = vb.p.numpy(), vb.q.numpy()
    d, rid = vb.draft_tokens.numpy(), vb.request_ids.numpy().view(np.uint32)
    T = max(1, min(T, n_req))
    bounds = [n_req * t // T for t in range(T + 1)]

    def lookup_part(t):
        lo, hi = bounds[t], bounds[t + 1]
        o = offs[lo:hi + 1]
        return oracle.lookup(ctx[o[0]:o[-1]], (o - o[0]).astype(offs.dtype), 1, 4, 5)

    parts = list(pool.map(lookup_part, range(T)))
    plen = np.concatenate([pl for _, pl in parts])
    ctx_len = np.diff(offs).astype(np.int32)
    oracle.choose_k(0.7, ctx_len, plen, 5, oracle.POLICY_PLD, synth.SPEC_DESK_TARGET, synth.SPEC_DESK_DRAFT,
                    pld_cost_ms=0.05)

    def verify_part(t):
        lo, hi = bounds[t], bounds[t + 1]
        r0, r1 = int(ro[lo]), int(ro[hi])
        q0, q1 = r0 - lo, r1 - hi
        na, _, _ = oracle.verify(p[r0:r1], q[q0:q1], (ro[lo:hi + 1] - r0).astype(ro.dtype), d[q0:q1], rid[lo:hi],
                                 seed, step, K_MAX)
        return na

    na = np.concatenate(list(pool.map(verify_part, range(T))))
    oracle.update(0.7, na, ro)
    return int((na + 1).sum())


def cpu_baseline(budget_s=12.0):
    """The oracle on the box's host cores (all of them: one thread per core over request ranges)."""
    import concurrent.futures as cf

    import synth
    data = cpu_data()
    T = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    with cf.ThreadPoolExecutor(max_workers=T) as pool:
        t0 = time.perf_counter()
        toks, steps = 0, 0
        while True:
            toks += oracle_step_threaded(synth.DEFAULT_SEED, steps, data, pool, T)
            steps += 1
            if time.perf_counter() - t0 > budget_s or steps >= 60:
                break
        el = time.perf_counter() - t0
    # the single-thread figure as well (first steps, bounded)
    t1 = time.perf_counter()
    toks1, steps1 = 0, 0
    while steps1 < 3 or time.perf_counter() - t1 < 2.0:
        toks1 += oracle_step_sample(B, synth.DEFAULT_SEED, steps1, data)
        steps1 += 1
        if steps1 >= 30:
            break
    el1 = time.perf_counter() - t1
    return {"value": toks / el, "unit": UNIT, "cores": T, "kind": "oracle",
            "sample": f"{steps} full steps of the bench workload (B={B}, V={V}) on {T} host threads "
                      f"(request ranges; {cpu_model()}), {el:.1f} s",
            "single_thread": {"value": toks1 / el1, "steps": steps1}}


def run_reference(args, rank, world):
    """The reference arm for this tier: the CPU oracle as it stands, on the box's host cores (request
    ranges on a thread pool, as cpu_baseline), each step a bounded sample of the workload."""
    if rank != 0:
        return None
    import concurrent.futures as cf

    import synth
    data = cpu_data()
    T = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    with cf.ThreadPoolExecutor(max_workers=T) as pool:
        # size the per-step sample so the whole run stays within ~2 minutes
        t0 = time.perf_counter()
        oracle_step_threaded(synth.DEFAULT_SEED, 0, data, pool, T)
        per_step = time.perf_counter() - t0
        total = max(1, args.steps + args.warmup)
        n_req = int(max(1, min(B, B * 100.0 / total / max(per_step, 1e-6))))
        for w in range(args.warmup):
            oracle_step_threaded(synth.DEFAULT_SEED, w, data, pool, T, n_req)
        t0 = time.perf_counter()
        toks = 0
        for s in range(args.steps):
            toks += oracle_step_threaded(synth.DEFAULT_SEED, args.warmup + s, data, pool, T, n_req)
        el = time.perf_counter() - t0
    value = toks / el
    sample = f"first {n_req} of {B} requests per step, {T} host threads over request ranges ({cpu_model()})"
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3 / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded, synth/)",
            "config": {"workload": WORKLOAD, "global_batch": B, "vocab": V, "k_max": K_MAX,
                       "ctx_len": L_CTX, "parallelism": f"cpu oracle, {T} threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": T, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


class nvtx_range:
    """torch.cuda.nvtx range around a bench phase when --nvtx is given (no-op otherwise)."""

    def __init__(self, args, name):
        self.on, self.name = bool(getattr(args, "nvtx", False)), name

    def __enter__(self):
        if self.on:
            import torch
            torch.cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *a):
        if self.on:
            import torch
            torch.cuda.nvtx.range_pop()


def main():
    # stdout carries only the JSON line: anything native code writes to fd 1 (e.g. NCCL's version
    # banner) is sent to stderr, and the line goes to a private duplicate of the original stdout
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    args = parse()
    if args.nvtx:
        os.environ["TSV_NVTX"] = "1"  # read once by libtsv at its first entry-point call
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), file=_JSON_OUT, flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(_dev_index(local_rank))
        if SHARED_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    runners = {"config4": run_config4, "greedy": run_greedy, "logits": run_logits, "config5": run_config5,
               "loop": run_loop, "strong": run_strong}
    if args.workload in runners:
        line = runners[args.workload](args, rank, world, local_rank)
        if line is not None:
            print(json.dumps(line), file=_JSON_OUT, flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return
    with nvtx_range(args, "bench:step"):
        line = run_ours(args, rank, world, local_rank)
    if not args.no_extras:
        # every other workload of BASELINE.json / SURVEY.md 8(f) as a sub-object of the one JSON line, each
        # timed the same way (its own CUDA events, roofline, clocks and device status)
        extras = {}
        plan = [("strong", run_strong, {})] if world > 1 else []
        plan += [("config4", run_config4, {"shard_mode": "auto"})]
        if world == 1:
            plan += [("config4_sharded_p2p", run_config4, {"shard_mode": "p2p"}),
                     ("config4_sharded_p2p_fused", run_config4, {"shard_mode": "p2p_fused"})]
        else:  # the other exchanges of config 4 over the N ranks (the "config4" line is the LL exchange)
            plan += [("config4_p2p_fused", run_config4, {"shard_mode": "p2p_fused"})]
            if not SHARED_GPU:  # NCCL cannot put two ranks on one GPU
                plan += [("config4_nccl_lazy", run_config4, {"shard_mode": "lazy"})]
        plan += [("greedy", run_greedy, {}), ("logits", run_logits, {}), ("config5", run_config5, {}),
                 ("loop", run_loop, {})]
        for name, fn, over in plan:
            a2 = argparse.Namespace(**vars(args))
            for k, v in over.items():
                setattr(a2, k, v)
            t0 = time.perf_counter()
            try:
                with nvtx_range(args, f"bench:{name}"):
                    sub = fn(a2, rank, world, local_rank)
            except Exception as e:  # noqa: BLE001  (a failed sub-workload must not hide the main line)
                sub = {"error": f"{type(e).__name__}: {e}"[:300]} if rank == 0 else None
            if sub is not None:
                sub["wall_s"] = round(time.perf_counter() - t0, 2)
                extras[name] = sub
        if line is not None:
            line["workloads"] = extras
    if line is not None:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), file=_JSON_OUT, flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
