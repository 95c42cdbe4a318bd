"""Host-side pieces of bench.py that run on CPU: the CPU baseline / reference arm run the oracle
over request ranges on a thread pool; the token counts must equal the single-thread step's."""
import concurrent.futures as cf

import bench
import synth


def test_threaded_oracle_step_equals_single_thread():
    data = bench.cpu_data()
    with cf.ThreadPoolExecutor(4) as pool:
        for step, n_req in ((0, 37), (3, 5), (7, 1)):
            a = bench.oracle_step_threaded(synth.DEFAULT_SEED, step, data, pool, 4, n_req)
            b = bench.oracle_step_sample(n_req, synth.DEFAULT_SEED, step, data)
            assert a == b, (step, n_req, a, b)


def test_verify_alg_bytes_matches_definition():
    # 4V (p row m) + 4V [m < k] (q row m, dense) + 32 B per tested gather (x2 dense)
    # + 4(k + 3) metadata + 4(k_max + 2) outputs, per request
    V, k_max = 100, 8
    m, k = [0, 3, 2], [0, 3, 5]
    want = 0
    for mi, ki in zip(m, k):
        rej = 1 if mi < ki else 0
        want += 4 * V * (1 + rej) + 32 * (mi + rej) * 2 + 4 * (ki + 3) + 4 * (k_max + 2)
    assert bench.verify_alg_bytes(m, k, True, V, k_max) == want
