"""CPU-side checks (no GPU): the C-ABI library loads and exports every entry point declared in
include/sfkv.h; its host-callable hash agrees with the oracle's independent restatement; the
oracle agrees with the reference's own functions (oracle/_ref/libsfref.so) on random inputs."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_lib
import paper_2603_13605_b200 as pkg
from paper_2603_13605_b200.abi import Config, Pool

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(REPO, "include", "sfkv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:sfkv|sfmm|sfmap|sfmet)_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = pkg.load_library()
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.sfkv_abi_version() == 2


def test_pool_create_without_gpu_fails_loudly():
    api = pkg.api()
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(Exception) as ei:
        pkg.Pool(api, pkg.Config())
    assert "ENODEV" in str(ei.value) or "ECUDA" in str(ei.value)


def test_block_hash_matches_oracle(oracle_api):
    lib = pkg.load_library()
    lib.sfkv_block_digest.restype = C.c_uint64
    lib.sfkv_block_digest.argtypes = [C.c_uint64, C.c_uint32, C.c_void_p]
    lib.sfkv_chain_finalize.restype = C.c_uint64
    lib.sfkv_chain_finalize.argtypes = [C.c_uint64]
    rng = np.random.default_rng(3)
    for _ in range(500):
        n = int(rng.integers(1, 17))
        k = int(rng.integers(0, 1 << 20))
        t = rng.integers(0, 1 << 32, size=16, dtype=np.uint64).astype(np.uint32)
        a = lib.sfkv_block_digest(k, n, t.ctypes.data)
        b = oracle_api.block_digest(k, n, t.ctypes.data)
        assert a == b
        s = int(rng.integers(0, 1 << 63))
        assert lib.sfkv_chain_finalize(s) == oracle_api.chain_finalize(s) >= 2


def test_golden_fixtures_present():
    import replay
    names = replay.stream_names()
    for n in ("support_demo", "chain_preserve", "chain_flush", "mapped_one_bit", "alt_pressure",
              "chain_scale"):
        assert n in names


# ---------------------------------------------------------------- oracle vs reference ----
ref = oracle_lib.load_ref()
needs_ref = pytest.mark.skipif(ref is None, reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
def test_oracle_pressure_matches_reference(oracle_api):
    """acceptance_tests.cpp:227-269 style: random trackers, seed 0x9E55, 1000 trials."""
    ref.sfref_pressure_actions.restype = C.c_int
    po = __import__("replay").default_pressure(oracle_api)
    rng = np.random.default_rng(0x9E55)
    for trial in range(1000):
        nb = int(rng.integers(1, 4))
        refs = [f"b{i}" for i in range(nb)]
        nwf = int(rng.integers(0, 12))
        names = [f"w{int(x)}" for x in rng.choice(1000, size=nwf, replace=False)]
        entries = [(w, b) for w in names for b in range(nb) if rng.random() < 0.6]
        n = len(entries)
        wf_c = (C.c_char_p * max(n, 1))(*[e[0].encode() for e in entries])
        backend = np.array([e[1] for e in entries], dtype=np.int32)
        ts = rng.integers(0, 5, size=n).astype(np.float64)
        inf = (rng.random(n) < 0.3).astype(np.int32)
        pres = (rng.random(n) < 0.8).astype(np.uint8)
        util = rng.choice([0.3, 0.85, 0.9], size=nb).astype(np.float64)
        refs_c = (C.c_char_p * nb)(*[r.encode() for r in refs])
        out_ref = np.zeros(nb, dtype=np.int64)
        ref.sfref_pressure_actions(C.c_longlong(n), wf_c, backend.ctypes.data_as(C.c_void_p),
                                   ts.ctypes.data_as(C.c_void_p), inf.ctypes.data_as(C.c_void_p),
                                   pres.ctypes.data_as(C.c_void_p), None, C.c_int(nb), refs_c,
                                   util.ctypes.data_as(C.c_void_p), C.c_double(0.85),
                                   out_ref.ctypes.data_as(C.c_void_p))
        order = sorted(set(names), key=lambda s: s.encode())
        rank = np.array([order.index(e[0]) for e in entries], dtype=np.uint32)
        got = po(backend, ts, rank, inf, pres, util, 0.85)
        np.testing.assert_array_equal(got, out_ref)


@needs_ref
def test_oracle_prefix_match_matches_reference(oracle_api):
    ref.sfref_pool_create.restype = C.c_void_p
    ref.sfref_complete.restype = C.c_longlong
    ref.sfref_complete.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_longlong, C.c_void_p]
    ref.sfref_batch_create.restype = C.c_void_p
    ref.sfref_batch_create.argtypes = [C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p]
    ref.sfref_prefix_match_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    ref.sfref_occupancy_tokens.restype = C.c_longlong
    ref.sfref_occupancy_tokens.argtypes = [C.c_void_p]
    from paper_2603_13605_b200.abi import Config, Pool, csr
    from scenarios import Workload
    n_wf = 40
    wl = Workload(9, n_wf, vocab=50)  # small vocab: many accidental matches
    h = ref.sfref_pool_create(C.c_longlong(5000))
    o = Pool(oracle_api, Config(max_workflows=n_wf, n_blocks=4000, capacity_tokens=5000,
                                max_pin_blocks=64))
    rng = np.random.default_rng(9)
    for step in range(6):
        wfs = rng.choice(n_wf, size=20, replace=False).astype(np.int32)
        seqs, off, tok = wl.batch(wfs)
        names = (C.c_char_p * len(wfs))(*[f"wf{w}".encode() for w in wfs])
        b = ref.sfref_batch_create(len(wfs), names, off.ctypes.data, tok.ctypes.data)
        m_ref = np.zeros(len(wfs), dtype=np.int64)
        ref.sfref_prefix_match_batch(h, b, m_ref.ctypes.data)
        np.testing.assert_array_equal(o.match(wfs, off, tok), m_ref)
        acc = C.c_int()
        for w, s in zip(wfs, seqs):
            arr = np.ascontiguousarray(s, dtype=np.uint32)
            ref.sfref_complete(h, f"wf{w}".encode(), arr.ctypes.data, len(arr), C.byref(acc))
        o.commit(wfs, off, tok)
        assert o.stats()["occupancy_tokens"] == ref.sfref_occupancy_tokens(h)


@needs_ref
def test_oracle_reroute_matches_reference(oracle_api):
    ref.sfref_reroute.restype = C.c_int
    ref.sfref_reroute.argtypes = [C.c_int, C.c_void_p, C.c_ulonglong]
    rng = np.random.default_rng(4)
    for _ in range(300):
        c = int(rng.integers(2, 6))
        depth = rng.integers(0, 6, size=c).astype(np.uint64)
        limit = int(rng.integers(1, 6))
        want = ref.sfref_reroute(c, depth.ctypes.data, limit)
        # the oracle's cost batch with candidate 0 forced as the primary and cyclic alternates
        P = np.array([0], np.int64)
        M = np.zeros(c, np.int64)
        O = np.array([0], np.int64)
        par = [np.array([0.0] + [1.0] * (c - 1)), np.zeros(c), np.zeros(c), np.zeros(c)]
        alt = np.full((c, c), -1, np.int32)
        alt[0, : c - 1] = np.arange(1, c)
        d = depth.copy()
        ch = np.zeros(1, np.int32)
        co = np.zeros(1, np.float64)
        oracle_api.check("cost", oracle_api.cost_batch(1, c, P.ctypes.data, M.ctypes.data,
                         O.ctypes.data, *[x.ctypes.data for x in par], alt.ctypes.data,
                         d.ctypes.data, limit, ch.ctypes.data, co.ctypes.data))
        assert ch[0] == want


@needs_ref
def test_oracle_threshold_matches_reference(oracle_api):
    ref.sfref_map_threshold.restype = C.c_int
    ref.sfref_map_threshold.argtypes = [C.c_double, C.c_double]
    rng = np.random.default_rng(11)
    s = np.concatenate([rng.normal(100, 30, 500), [100.0, 99.999999, 100.000001]])
    out = np.zeros(len(s), np.int32)
    oracle_api.check("thr", oracle_api.threshold_batch(len(s), s.ctypes.data, 100.0, out.ctypes.data))
    for x, o in zip(s, out):
        assert (o == 0) == bool(ref.sfref_map_threshold(float(x), 100.0))


def test_oracle_hashes_full_c2_size_fast(oracle_api):
    """The oracle's chained hashes for the full C2 batch (10k requests, 1.78 M blocks) in seconds:
    the checker of tests/test_gpu_parity.py::test_full_c2_size_match."""
    import time
    import bench
    wl = bench.make_workload(0x0A1A + 1, 10_000)
    n = wl["n"]
    o = Pool(oracle_api, Config(max_workflows=n, n_blocks=1024, capacity_tokens=1 << 40,
                                max_pin_blocks=int(bench.blocks_of(wl["req_len"]).max()) + 1, table_log2=12))
    t0 = time.perf_counter()
    M, h = o.match(np.arange(n, dtype=np.int32), wl["req_off"], wl["req_tok"], want_hash=True)
    assert time.perf_counter() - t0 < 60
    assert (M == 0).all() and len(h) == int(bench.blocks_of(wl["req_len"]).sum())
