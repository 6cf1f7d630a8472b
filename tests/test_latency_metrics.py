"""Batched latency model and TTFT percentiles (§8f-3).

CPU: the oracle restatement equals the reference's own SimulatedBackend timing (queue, ttft, total
of every CompletionResponse, simulated_backend.cpp:72-133) for requests queued behind each other
on one backend with pinned-prefix hits, and the reference's percentile_nearest_rank
(metrics.cpp:22-28) for every percentile 0..100, bit for bit. GPU (`-m gpu`): sfmet_* equal the
oracle bit for bit on large random batches (no FMA contraction in the kernel)."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2603_13605_b200.abi import latency_batch, nearest_rank

REF_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "libsfref.so")


def _ref():
    L = C.CDLL(REF_LIB)
    L.sfref_sim_timing.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_longlong, C.c_int,
                                   C.POINTER(C.c_char_p), C.POINTER(C.c_char_p)] + [C.c_void_p] * 6
    L.sfref_percentile.restype = C.c_double
    L.sfref_percentile.argtypes = [C.c_longlong, C.c_void_p, C.c_int]
    return L


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_latency_matches_reference_backend(oracle_api, seed):
    L = _ref()
    rng = np.random.default_rng(seed)
    prefill, decode, overhead = [0.05, 1.0, 2.0][seed - 1], [1.0, 10.0, 0.3][seed - 1], [0.0, 7.5, 0.1][seed - 1]
    n, out_tokens = 40, int(rng.integers(0, 50))
    base = ["w%d" % i for i in range(6)]
    texts, wfs, ctx = [], [], {}
    for i in range(n):
        w = str(rng.choice(base + [""]))  # "" = an unpinned routing call
        prev = ctx.get(w, [])
        toks = prev + ["t%d" % x for x in rng.integers(0, 30, size=int(rng.integers(0, 40)))]
        if w and rng.random() < 0.3 and toks:
            toks[int(rng.integers(0, len(toks)))] = "zz"  # a rewrite: partial hit
        ctx[w] = toks
        texts.append(" ".join(toks).encode())
        wfs.append(w.encode())
    q, tt, tot = (np.zeros(n) for _ in range(3))
    P, M, O = (np.zeros(n, np.int64) for _ in range(3))
    L.sfref_sim_timing(prefill, decode, overhead, 2, out_tokens, n, (C.c_char_p * n)(*wfs), (C.c_char_p * n)(*texts),
                       *[a.ctypes.data for a in (q, tt, tot, P, M, O)])
    assert (q > 0).any() and (M > 0).any()  # queueing and cache hits both exercised
    ttft, total, svc = latency_batch(oracle_api, np.zeros(n, np.int32), q, P, M, O, [overhead], [prefill], [decode])
    assert ttft.tobytes() == tt.tobytes()
    assert total.tobytes() == tot.tobytes()


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
@pytest.mark.parametrize("n", [1, 2, 7, 99, 100, 101, 1000])
def test_oracle_nearest_rank_matches_reference(oracle_api, n):
    L = _ref()
    rng = np.random.default_rng(n)
    x = np.round(rng.exponential(100.0, size=n), 3)  # ties included
    s = np.sort(x)
    pct = np.arange(0, 101, dtype=np.int32)
    want = np.array([L.sfref_percentile(n, s.ctypes.data, int(p)) for p in pct])
    assert nearest_rank(oracle_api, x, pct).tobytes() == want.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 1000, 300_000])
def test_gpu_latency_and_percentiles_match_oracle(gpu_api, oracle_api, n):
    rng = np.random.default_rng(n)
    nb = 8
    b = rng.integers(0, nb, size=n)
    P = rng.integers(0, 200_000, size=n)
    M = (P * rng.random(n)).astype(np.int64)
    O = rng.integers(0, 4096, size=n)
    q = rng.exponential(50.0, size=n)
    par = [rng.random(nb) * s for s in (20.0, 2.0, 30.0)]
    got = latency_batch(gpu_api, b, q, P, M, O, *par)
    want = latency_batch(oracle_api, b, q, P, M, O, *par)
    for g, w in zip(got, want):
        assert g.tobytes() == w.tobytes()
    pct = np.arange(0, 101, dtype=np.int32)
    assert nearest_rank(gpu_api, got[0], pct).tobytes() == nearest_rank(oracle_api, want[0], pct).tobytes()
