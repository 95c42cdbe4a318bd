"""CPU-only checks of the C ABI: libtsv.so loads, exports every symbol include/tsv.h
declares, the ctypes mirrors match the C layouts (gcc-compiled offsetof probe), and
host-side validation rejects bad arguments before any launch (no GPU needed)."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "tsv.h")


@pytest.fixture(scope="module")
def tsv():
    from paper_2406_14066_b200 import build
    build.build()
    from paper_2406_14066_b200 import tsv as t
    return t


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^TSV_API\s+[\w\s\*]+?\b(tsv_\w+)\s*\(", txt, flags=re.M)))


def test_every_declared_symbol_exported(tsv):
    syms = declared_symbols()
    assert len(syms) >= 16
    out = subprocess.run(["nm", "-D", "--defined-only", tsv.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tsv_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(tsv.EXPORTED) == syms
    for s in syms:
        assert getattr(tsv.lib(), s) is not None


def test_abi_version(tsv):
    assert tsv.tsv_abi_version() == 2


PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "tsv.h"
#define F(T, m) printf(#T " " #m " %zu\n", offsetof(T, m));
int main(void) {
  printf("tsv_verify_args sizeof %zu\n", sizeof(tsv_verify_args));
  F(tsv_verify_args, p) F(tsv_verify_args, q) F(tsv_verify_args, row_offsets)
  F(tsv_verify_args, draft_tokens) F(tsv_verify_args, request_ids) F(tsv_verify_args, num_accepted)
  F(tsv_verify_args, out_tokens) F(tsv_verify_args, device_status) F(tsv_verify_args, workspace)
  F(tsv_verify_args, workspace_bytes) F(tsv_verify_args, ld) F(tsv_verify_args, seed)
  F(tsv_verify_args, step) F(tsv_verify_args, B) F(tsv_verify_args, k_max) F(tsv_verify_args, rows_p)
  F(tsv_verify_args, vocab) F(tsv_verify_args, vocab_offset) F(tsv_verify_args, vocab_global)
  F(tsv_verify_args, chunk) F(tsv_verify_args, flags) F(tsv_verify_args, step_counts)
  printf("tsv_shard_tuple sizeof %zu\n", sizeof(tsv_shard_tuple));
  printf("tsv_latency_model sizeof %zu\n", sizeof(tsv_latency_model));
  return 0;
}
"""


def test_ctypes_layout_matches_c(tsv):
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "probe.c")
        exe = os.path.join(d, "probe")
        open(src, "w").write(PROBE)
        subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    c = {}
    for line in out:
        if line.strip():
            t, m, v = line.split()
            c[(t, m)] = int(v)
    assert c[("tsv_verify_args", "sizeof")] == ctypes.sizeof(tsv.VerifyArgs)
    for name, _ in tsv.VerifyArgs._fields_:
        assert c[("tsv_verify_args", name)] == getattr(tsv.VerifyArgs, name).offset, name
    assert c[("tsv_shard_tuple", "sizeof")] == tsv.SHARD_TUPLE_BYTES
    assert c[("tsv_latency_model", "sizeof")] == ctypes.sizeof(tsv.LatencyModel)


def test_host_validation_without_gpu(tsv):
    L = tsv.lib()
    # bad n-gram range: rejected before any device work
    assert L.tsv_propose_lookup(None, None, 4, 3, 2, 5, None, None, None, None) == 1
    assert b"n_min" in L.tsv_last_error()
    assert L.tsv_propose_lookup(None, None, -1, 1, 2, 5, None, None, None, None) == 1
    # B = 0 is a no-op
    assert L.tsv_propose_lookup(None, None, 0, 1, 2, 5, None, None, None, None) == 0
    # the flagged entry points: unknown flag bits are rejected before any device work
    assert L.tsv_propose_lookup_ex(None, None, 0, 1, 2, 5, None, None, None, tsv.LOOKUP_INPUTS_READY, None) == 0
    assert L.tsv_propose_lookup_ex(None, None, 4, 1, 2, 5, None, None, None, 2, None) == 1
    assert b"flags" in L.tsv_last_error()
    m0 = tsv.LatencyModel(0.001, 0.05, 2.0)
    assert L.tsv_propose_lookup_choose_k_ex(None, None, 4, 1, 4, 5, None, None, None, 0, None, m0, 0.05, -1, None,
                                            None, None, None, None, None, 6, None) == 1
    assert b"flags" in L.tsv_last_error()
    a = tsv.VerifyArgs()
    a.B, a.k_max = 4, 16
    assert L.tsv_verify_accept(ctypes.byref(a), None) == 1
    assert b"k_max" in L.tsv_last_error()
    a.k_max = 4
    assert L.tsv_verify_accept(ctypes.byref(a), None) == 1  # NULL arrays
    assert L.tsv_verify_accept(None, None) == 1
    assert L.tsv_update_acceptance(None, 0, None, None, 3, 1.5, 0, None) == 1
    assert b"decay" in L.tsv_last_error()
    m = tsv.LatencyModel(0.001, 0.05, 2.0)
    assert L.tsv_goodput_choose_k(None, 0, None, None, 0, 8, 0, m, m, 0.0, -1, None, None, None, None) == 1
    assert L.tsv_goodput_choose_k(None, 0, None, None, 4, 8, 7, m, m, 0.0, -1, None, None, None, None) == 1
    assert b"policy" in L.tsv_last_error()


def test_binding_rejects_cpu_tensors(tsv):
    import torch
    with pytest.raises(ValueError):
        tsv._ptr(torch.zeros(4))


def test_empty_batch_is_a_noop_without_device_work(tsv):
    # B = 0: every entry point returns TSV_OK before touching the device (no GPU needed)
    L = tsv.lib()
    a = tsv.VerifyArgs()
    a.B, a.k_max, a.vocab, a.vocab_global, a.ld = 0, 4, 8, 8, 8
    dummy = ctypes.c_void_p(16)
    assert L.tsv_verify_accept(ctypes.byref(a), None) == 0
    assert L.tsv_verify_greedy(ctypes.byref(a), None) == 0
    assert L.tsv_verify_accept_logits(ctypes.byref(a), 1.0, None) == 0
    assert L.tsv_verify_accept_update(ctypes.byref(a), dummy, 0, 0.9, 0, None) == 0
    assert L.tsv_verify_shard_partial(ctypes.byref(a), None, None) == 0
    assert L.tsv_verify_shard_combine(ctypes.byref(a), None, 1, None) == 0
    assert L.tsv_verify_shard_flags(ctypes.byref(a), None, None) == 0
    assert L.tsv_verify_shard_race(ctypes.byref(a), None, None, None) == 0
    assert L.tsv_verify_shard_emit(ctypes.byref(a), None, None, None) == 0
    assert L.tsv_update_acceptance(None, 0, None, None, 0, 0.9, 0, None) == 0
    assert L.tsv_sim_target(None, 5, None, 0, None, 16, 16, 0, None, None, None, None, None) == 0
    assert L.tsv_context_append(None, 16, 0, None, None, 5, None, None, None) == 0
    assert L.tsv_softmax_rows(None, 16, 16, 0, 1.0, None, None) == 0
    m = tsv.LatencyModel(0.001, 0.05, 2.0)
    assert L.tsv_goodput_choose_k_batched(None, None, None, None, 0, 8, 0, m, m, 0.0, -1, None, None, None, None) == 0


def test_workspace_errors_return_tsv_err_workspace(tsv):
    # a NULL or too small workspace is TSV_ERR_WORKSPACE (5), checked on the host before any launch
    L = tsv.lib()
    buf = ctypes.create_string_buffer(64 * 1024 + 16)
    base = (ctypes.addressof(buf) + 15) // 16 * 16  # host addresses: validation never dereferences them
    a = tsv.VerifyArgs()
    a.B, a.k_max, a.rows_p, a.vocab, a.vocab_global, a.ld = 4, 4, 20, 64, 64, 64
    for f in ("p", "q", "row_offsets", "draft_tokens", "request_ids", "num_accepted", "out_tokens"):
        setattr(a, f, base)
    need = ctypes.c_size_t(0)
    assert L.tsv_verify_workspace_size(ctypes.byref(a), ctypes.byref(need)) == 0 and need.value > 0
    a.workspace, a.workspace_bytes = None, 0
    assert L.tsv_verify_accept(ctypes.byref(a), None) == 5
    assert b"workspace" in L.tsv_last_error()
    a.workspace, a.workspace_bytes = base, need.value - 1
    assert L.tsv_verify_accept(ctypes.byref(a), None) == 5
    assert L.tsv_verify_accept_update(ctypes.byref(a), base, 0, 0.9, 0, None) == 5
    assert L.tsv_verify_greedy(ctypes.byref(a), None) == 5
    assert L.tsv_verify_shard_partial(ctypes.byref(a), base, None) == 5
    assert L.tsv_verify_shard_race(ctypes.byref(a), base, base, None) == 5
    m = tsv.LatencyModel(0.001, 0.05, 2.0)
    assert L.tsv_propose_lookup_choose_k(base, base, 4, 1, 4, 5, base, base, base, 0, base, m, 0.05, -1, base,
                                         None, None, None, None, None) == 5
    assert tsv.STATUS_NAMES[5] == "TSV_ERR_WORKSPACE"


def test_devstatus_bits_match_header(tsv):
    txt = open(HDR).read()
    bits = dict((n, int(v)) for n, v in re.findall(r"#define TSV_DEVSTATUS_(\w+) (\d+)u", txt))
    assert bits == {"BAD_TOKEN": tsv.DEVSTATUS_BAD_TOKEN, "BAD_K": tsv.DEVSTATUS_BAD_K,
                    "NO_WEIGHT": tsv.DEVSTATUS_NO_WEIGHT, "P2P_TIMEOUT": tsv.DEVSTATUS_P2P_TIMEOUT,
                    "BAD_CONTEXT": tsv.DEVSTATUS_BAD_CONTEXT, "WAIT_TIMEOUT": tsv.DEVSTATUS_WAIT_TIMEOUT}
