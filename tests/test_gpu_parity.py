"""GPU parity: libsfkv.so (sm_100a kernels behind the C ABI) against the CPU oracle and the
reference's own golden streams. Integer/index outputs must be bit-exact; KV payload bytes must be
byte-identical; mapper costs are compared as exact doubles (the kernels avoid FMA contraction),
well inside north_star's 1e-6 relative tolerance."""
import ctypes as C

import numpy as np
import pytest

import replay
from paper_2603_13605_b200.abi import BLOCK_TOKENS, Config, Pool, csr
from scenarios import Workload

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- Class A: golden replays ----
@pytest.mark.parametrize("name", replay.stream_names())
@pytest.mark.parametrize("batched", [False, True])
def test_gpu_replays_reference_stream(gpu_api, name, batched):
    lines = replay.load_stream(name)
    assert replay.replay(lines, gpu_api, batched=batched) > 0


# ---------------------------------------------------------------- Class B: vs the oracle -----
def _pair(gpu_api, oracle_api, cfg):
    return Pool(gpu_api, cfg), Pool(oracle_api, cfg)


def _assert_same_state(g, o, wfs):
    sg, so = g.stats(), o.stats()
    for k in ("occupancy_tokens", "capacity_rejections", "blocks_in_use", "table_live"):
        assert sg[k] == so[k], (k, sg[k], so[k])
    np.testing.assert_array_equal(g.refcounts(), o.refcounts())
    for w in wfs:
        ig, hg = g.pin_blocks(w)
        io, ho = o.pin_blocks(w)
        np.testing.assert_array_equal(ig, io)
        np.testing.assert_array_equal(hg, ho)
        assert g.pinned_token_count(w) == o.pinned_token_count(w)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_match_commit_flush_random(gpu_api, oracle_api, seed):
    n_wf = 96
    wl = Workload(seed, n_wf, n_sys=3, sys_len=(16, 80), ctx_len=(0, 70), append=(0, 50))
    cfg = Config(max_workflows=n_wf, n_blocks=6000, capacity_tokens=60_000, max_pin_blocks=64,
                 table_log2=14)
    g, o = _pair(gpu_api, oracle_api, cfg)
    rng = np.random.default_rng(seed + 100)
    for step in range(12):
        wfs = rng.choice(n_wf, size=int(rng.integers(1, n_wf)), replace=False).astype(np.int32)
        seqs, off, tok = wl.batch(wfs)
        Mg, hg = g.match(wfs, off, tok, want_hash=True)
        Mo, ho = o.match(wfs, off, tok, want_hash=True)
        np.testing.assert_array_equal(Mg, Mo)
        np.testing.assert_array_equal(hg, ho)
        bg, htg = g.lookup(off, tok)
        bo, hto = o.lookup(off, tok)
        np.testing.assert_array_equal(bg, bo)
        np.testing.assert_array_equal(htg, hto)
        sg = g.commit(wfs, off, tok)
        so = o.commit(wfs, off, tok)
        np.testing.assert_array_equal(sg, so)
        if step % 4 == 3:
            fl = rng.choice(n_wf, size=8, replace=False).astype(np.int32)
            np.testing.assert_array_equal(g.flush_batch(fl), o.flush_batch(fl))
        _assert_same_state(g, o, range(n_wf))
    assert g.flush(-1) == o.flush(-1)
    _assert_same_state(g, o, range(n_wf))


def test_capacity_rejections_and_edge_lengths(gpu_api, oracle_api):
    cfg = Config(max_workflows=8, n_blocks=512, capacity_tokens=100, max_pin_blocks=16)
    g, o = _pair(gpu_api, oracle_api, cfg)
    seqs = [[], [7] * 15, [7] * 16, [7] * 17, list(range(1, 61)), list(range(1, 81))]
    wfs = np.arange(len(seqs), dtype=np.int32)
    off, tok = csr(seqs)
    np.testing.assert_array_equal(g.commit(wfs, off, tok), o.commit(wfs, off, tok))
    _assert_same_state(g, o, range(8))
    np.testing.assert_array_equal(g.match(wfs, off, tok), o.match(wfs, off, tok))
    assert g.preserve(0) and o.preserve(0)  # an empty pin counts as present
    assert g.cache_utilization() == o.cache_utilization()


def test_reference_known_answers(gpu_api):
    """test_backend_sim.cpp:89-103 (LCP) and 134-144 (capacity) on the GPU pool."""
    g = Pool(gpu_api, Config(max_workflows=4, n_blocks=64, capacity_tokens=100, max_pin_blocks=8))
    a, b, c, d, e, x, y = 1, 2, 3, 4, 5, 6, 7
    off, tok = csr([[a, b, c]])
    assert g.commit(np.array([0], np.int32), off, tok)[0] == 1
    for seq, want, wf in (([a, b, c, d, e], 3, 0), ([x, y], 0, 0), ([a, b, c], 0, 1)):
        o2, t2 = csr([seq])
        assert g.match(np.array([wf], np.int32), o2, t2)[0] == want
    g2 = Pool(gpu_api, Config(max_workflows=4, n_blocks=64, capacity_tokens=100, max_pin_blocks=8))
    st = g2.commit(np.array([0, 1], np.int32), *csr([[1] * 60, [2] * 80]))
    assert list(st) == [1, 0] and g2.stats()["capacity_rejections"] == 1
    assert g2.flush(0) == 60 and g2.flush(0) == 0


def test_payload_scatter_cow_gather(gpu_api, oracle_api):
    torch = pytest.importorskip("torch")
    n_wf = 24
    cfg = Config(max_workflows=n_wf, n_blocks=1500, capacity_tokens=50_000, max_pin_blocks=40,
                 table_log2=12, n_slabs=4, slab_row_bytes=32)
    g, o = _pair(gpu_api, oracle_api, cfg)
    wl = Workload(7, n_wf, n_sys=2, sys_len=(16, 48), ctx_len=(0, 40), append=(1, 30))
    rng = np.random.default_rng(7)
    row = cfg.slab_row_bytes
    for step in range(6):
        wfs = rng.choice(n_wf, size=int(rng.integers(1, n_wf)), replace=False).astype(np.int32)
        seqs, off, tok = wl.batch(wfs)
        M = o.match(wfs, off, tok)
        np.testing.assert_array_equal(g.match(wfs, off, tok), M)
        # staging rows [M, P) per request: [slab][P-M][row]
        sizes = [cfg.n_slabs * (len(s) - int(m)) * row for s, m in zip(seqs, M)]
        kv_off = np.zeros(len(seqs), dtype=np.int64)
        kv_off[1:] = np.cumsum(sizes)[:-1]
        staging = rng.integers(0, 256, size=max(int(sum(sizes)), 16), dtype=np.uint8)
        st_o = o.commit(wfs, off, tok, kv_src=staging, kv_src_off=kv_off, m_expected=M)
        dev = torch.from_numpy(staging).cuda()
        st_g = g.commit(wfs, off, tok, kv_src=dev, kv_src_off=kv_off, m_expected=M)
        np.testing.assert_array_equal(st_g, st_o)
        _assert_same_state(g, o, range(n_wf))
        # gather every pinned workflow and compare bytes
        lens = [o.pinned_token_count(w) for w in range(n_wf)]
        dst_off = np.zeros(n_wf, dtype=np.int64)
        dst_off[1:] = np.cumsum([cfg.n_slabs * L * row for L in lens])[:-1]
        total = int(sum(cfg.n_slabs * L * row for L in lens)) + 16
        ho = np.zeros(total, dtype=np.uint8)
        allw = np.arange(n_wf, dtype=np.int32)
        oracle_api.check("gather", oracle_api.gather(o.h, n_wf, allw.ctypes.data, ho.ctypes.data,
                                                     dst_off.ctypes.data))
        dg = torch.zeros(total, dtype=torch.uint8, device="cuda")
        dw = torch.from_numpy(allw).cuda()
        doff = torch.from_numpy(dst_off).cuda()
        gpu_api.check("gather_dev", gpu_api.gather_dev(g.h, n_wf, C.c_void_p(dw.data_ptr()),
                                                       C.c_void_p(dg.data_ptr()),
                                                       C.c_void_p(doff.data_ptr())))
        gpu_api.check("pool_sync", gpu_api.pool_sync(g.h))
        np.testing.assert_array_equal(dg.cpu().numpy(), ho)


def test_stale_payload_commit_is_refused(gpu_api):
    torch = pytest.importorskip("torch")
    cfg = Config(max_workflows=4, n_blocks=64, capacity_tokens=1000, max_pin_blocks=8, n_slabs=2,
                 slab_row_bytes=16)
    g = Pool(gpu_api, cfg)
    off, tok = csr([[1, 2, 3]])
    stg = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(Exception):
        g.commit(np.array([0], np.int32), off, tok, kv_src=stg, kv_src_off=np.zeros(1, np.int64),
                 m_expected=np.array([2], np.int64))
    assert g.stats()["occupancy_tokens"] == 0


def test_handoff_between_pools(gpu_api, oracle_api):
    cfg = Config(max_workflows=8, n_blocks=400, capacity_tokens=10_000, max_pin_blocks=32,
                 table_log2=10, n_slabs=2, slab_row_bytes=16)
    ga, gb = Pool(gpu_api, cfg), Pool(gpu_api, cfg)
    oa, ob = Pool(oracle_api, cfg), Pool(oracle_api, cfg)
    rng = np.random.default_rng(5)
    seqs = [rng.integers(1, 1000, size=n).astype(np.uint32) for n in (70, 33, 16)]
    wfs = np.arange(3, dtype=np.int32)
    off, tok = csr(seqs)
    sizes = [cfg.n_slabs * len(s) * cfg.slab_row_bytes for s in seqs]
    kv_off = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    staging = rng.integers(0, 256, size=int(sum(sizes)), dtype=np.uint8)
    import torch
    for (p, stg) in ((ga, torch.from_numpy(staging).cuda()), (oa, staging)):
        p.commit(wfs, off, tok, kv_src=stg, kv_src_off=kv_off)
    # pre-existing partial pin on the destination for wf 5 (COW source on the dst side)
    o5, t5 = csr([seqs[0][:40]])
    for p in (gb, ob):
        p.commit(np.array([5], np.int32), o5, t5)
    for src_wf, dst_wf in ((0, 5), (1, 1), (2, 2)):
        assert ga.handoff_to(src_wf, gb, dst_wf) == oa.handoff_to(src_wf, ob, dst_wf)
    _assert_same_state(gb, ob, range(8))


# ---------------------------------------------------------------- K6 / K7 ----------------
def test_pressure_argmin_random(gpu_api, oracle_api):
    rng = np.random.default_rng(1234)  # test_memory.cpp:131-175 uses seed 1234, 300 trials
    pg = replay.default_pressure(gpu_api)
    po = replay.default_pressure(oracle_api)
    for trial in range(300):
        nb = int(rng.integers(1, 5))
        n = int(rng.integers(0, 60))
        backend = rng.integers(0, nb, size=n).astype(np.int32)
        ts = rng.integers(0, 8, size=n).astype(np.float64)  # many ties
        wr = rng.permutation(n).astype(np.uint32)
        inf = (rng.random(n) < 0.3).astype(np.int32) * rng.integers(1, 3, size=n).astype(np.int32)
        pres = (rng.random(n) < 0.8).astype(np.uint8)
        util = rng.choice([0.5, 0.85, 0.86, 1.0], size=nb).astype(np.float64)
        np.testing.assert_array_equal(pg(backend, ts, wr, inf, pres, util, 0.85),
                                      po(backend, ts, wr, inf, pres, util, 0.85))


@pytest.mark.parametrize("nb,n,layout", [(8, 40_000, "backend_major"), (8, 40_000, "interleaved"),
                                         (40, 200_000, "random"), (100, 50_000, "random")])
def test_pressure_argmin_large(gpu_api, oracle_api, nb, n, layout):
    """The single-pass segmented kernel (<= 64 backends: warps of one backend reduce in one
    shuffle tree, mixed warps once per distinct backend) and the per-backend-pass fallback
    (> 64 backends) at tracker scale, against the oracle."""
    rng = np.random.default_rng(nb * 7 + n)
    if layout == "backend_major":
        backend = np.repeat(np.arange(nb, dtype=np.int32), n // nb)
    elif layout == "interleaved":  # the tracker's dense (workflow, backend) order
        backend = np.tile(np.arange(nb, dtype=np.int32), n // nb)
    else:
        backend = rng.integers(0, nb, size=n).astype(np.int32)
    n = len(backend)
    ts = np.round(rng.uniform(0, 50, n), 0)  # heavy ties: the rank tie-break decides
    wr = rng.permutation(n).astype(np.uint32)
    inf = (rng.random(n) < 0.2).astype(np.int32)
    pres = (rng.random(n) < 0.7).astype(np.uint8)
    util = rng.choice([0.5, 0.86, 1.0], size=nb).astype(np.float64)
    got = replay.default_pressure(gpu_api)(backend, ts, wr, inf, pres, util, 0.85)
    want = replay.default_pressure(oracle_api)(backend, ts, wr, inf, pres, util, 0.85)
    np.testing.assert_array_equal(got, want)
    assert (got >= 0).sum() == (util > 0.85).sum()


def _cost(api, dev, n, c, P, M, O, par, alt, depth, limit):
    choice = np.zeros(n, dtype=np.int32)
    cost = np.zeros(n, dtype=np.float64)
    args = [n, c, P.ctypes.data, M.ctypes.data, O.ctypes.data] + [x.ctypes.data for x in par] + \
           [alt.ctypes.data if alt is not None else None, depth.ctypes.data, limit,
            choice.ctypes.data, cost.ctypes.data]
    api.check("cost_batch", api.dev_call("cost_batch", dev, *args))
    return choice, cost


@pytest.mark.parametrize("limit", [0, 3, 40])
def test_mapper_cost_and_reroute(gpu_api, oracle_api, limit):
    rng = np.random.default_rng(11)
    n, c = 5000, 8
    P = rng.integers(1, 4096, size=n).astype(np.int64)
    M = (rng.random((n, c)) * P[:, None]).astype(np.int64).reshape(-1)
    O = rng.integers(0, 512, size=n).astype(np.int64)
    par = [rng.random(c) * 50, rng.random(c) * 2, rng.random(c) * 20, rng.random(c)]
    alt = np.full((c, c), -1, dtype=np.int32)
    for i in range(c):
        alt[i, : c - 1] = [(i + j) % c for j in range(1, c)]
    d0 = rng.integers(0, 5, size=c).astype(np.uint64)
    dg, do = d0.copy(), d0.copy()
    cg, kg = _cost(gpu_api, 0, n, c, P, M, O, par, alt, dg, limit)
    co, ko = _cost(oracle_api, 0, n, c, P, M, O, par, alt, do, limit)
    np.testing.assert_array_equal(cg, co)
    np.testing.assert_array_equal(kg, ko)  # exact doubles
    np.testing.assert_array_equal(dg, do)


@pytest.mark.parametrize("c", [8, 12, 20])  # the window pass for c <= 8 / <= 16, the warp walk above
@pytest.mark.parametrize("limit", [0, 3, 40, 700])
def test_mapper_device_entry_matches_oracle(gpu_api, oracle_api, limit, c):
    """sfmap_cost_batch_dev (device pointers, one stream) and sfmap_cost_batch both equal the
    oracle over 20k requests (many reroute windows, every candidate saturating at limit 700)."""
    import torch
    rng = np.random.default_rng(limit + 5 + c)
    n = 20_000
    P = rng.integers(1, 4096, size=n).astype(np.int64)
    M = (rng.random((n, c)) * P[:, None]).astype(np.int64).reshape(-1)
    O = rng.integers(0, 512, size=n).astype(np.int64)
    par = [rng.random(c) * 50, rng.random(c) * 2, rng.random(c) * 20, rng.random(c)]
    alt = np.full((c, c), -1, dtype=np.int32)
    for i in range(c):
        alt[i, : c - 1] = [(i + j) % c for j in range(1, c)]
    d0 = rng.integers(0, 5, size=c).astype(np.uint64)
    dh, do = d0.copy(), d0.copy()
    ch, co = _cost(gpu_api, 0, n, c, P, M, O, par, alt, dh, limit)
    cho, coo = _cost(oracle_api, 0, n, c, P, M, O, par, alt, do, limit)
    np.testing.assert_array_equal(ch, cho)
    np.testing.assert_array_equal(co, coo)
    np.testing.assert_array_equal(dh, do)
    t = {k: torch.from_numpy(v).cuda() for k, v in dict(P=P, M=M, O=O, alt=alt, d=d0.view(np.int64),
                                                          oh=par[0], pf=par[1], dc=par[2], qp=par[3]).items()}
    och = torch.zeros(n, dtype=torch.int32, device="cuda")
    oco = torch.zeros(n, dtype=torch.float64, device="cuda")
    ptr = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    gpu_api.check("cost_batch_dev", gpu_api.cost_batch_dev(
        0, n, c, ptr(t["P"]), ptr(t["M"]), ptr(t["O"]), ptr(t["oh"]), ptr(t["pf"]), ptr(t["dc"]), ptr(t["qp"]),
        ptr(t["alt"]), ptr(t["d"]), limit, ptr(och), ptr(oco), None))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(och.cpu().numpy(), ch)
    np.testing.assert_array_equal(oco.cpu().numpy(), co)
    np.testing.assert_array_equal(t["d"].cpu().numpy().view(np.uint64), dh)


def test_threshold_mapper(gpu_api, oracle_api):
    """test_mapper.cpp:54-89: 80 -> light, 100 -> light (tie), 5000 -> heavy at threshold 100."""
    s = np.array([80, 100, 5000, 100.0000001, -1, 0], dtype=np.float64)
    out = np.zeros(len(s), dtype=np.int32)
    gpu_api.check("threshold", gpu_api.threshold_batch(0, len(s), s.ctypes.data, 100.0, out.ctypes.data))
    assert list(out) == [0, 0, 1, 1, 0, 0]


def test_pool_exhaustion_aborts_batch_cleanly(gpu_api, oracle_api):
    """A commit that needs more physical blocks than are free fails with SFKV_EPOOL and leaves
    occupancy, pins and refcounts unchanged; the pool keeps working afterwards."""
    cfg = Config(max_workflows=8, n_blocks=10, capacity_tokens=10_000, max_pin_blocks=16,
                 table_log2=8)
    g = Pool(gpu_api, cfg)
    off, tok = csr([list(range(1, 100))])  # 7 blocks
    assert g.commit(np.array([0], np.int32), off, tok)[0] == 1
    before = (g.stats(), g.refcounts().copy(), g.pin_blocks(0)[0].copy())
    off2, tok2 = csr([list(range(500, 600))])  # 7 more blocks: only 3 free
    with pytest.raises(Exception) as ei:
        g.commit(np.array([1], np.int32), off2, tok2)
    assert "EPOOL" in str(ei.value)
    after = (g.stats(), g.refcounts(), g.pin_blocks(0)[0])
    assert after[0]["occupancy_tokens"] == before[0]["occupancy_tokens"]
    assert after[0]["capacity_rejections"] == before[0]["capacity_rejections"]
    np.testing.assert_array_equal(after[1], before[1])
    np.testing.assert_array_equal(after[2], before[2])
    assert g.flush(0) == 99
    assert g.commit(np.array([1], np.int32), off2, tok2)[0] == 1  # the abandoned claims heal
    assert g.match(np.array([1], np.int32), off2, tok2)[0] == 100
    lk, hit = g.lookup(off2, tok2)
    assert hit[0] == 96 and (lk[:6] >= 0).all()


def _c2_full():
    import bench
    return bench, bench.make_workload(0x0A1A + 1, 10_000)


def test_full_c2_size_match(gpu_api, oracle_api):
    """BASELINE configs[1] at full size (10k workflows, 1.7 M pinned blocks, 1.78 M request blocks):
    M equals the construction's known LCP (a size-independent property: append-only prompts match
    their whole pin, rewritten ones stop at the rewrite) and every chained block hash equals the
    oracle's."""
    bench, wl = _c2_full()
    n = wl["n"]
    mpb = int(bench.blocks_of(wl["req_len"]).max()) + 1
    nb = int(bench.blocks_of(wl["base"]).sum()) + 2 * mpb + 1024
    g = Pool(gpu_api, Config(max_workflows=n, n_blocks=nb, capacity_tokens=1 << 50, max_pin_blocks=mpb,
                             table_log2=int(np.ceil(np.log2(2 * nb))) + 1))
    wf = np.arange(n, dtype=np.int32)
    for c0 in range(0, n, 2000):
        c1 = min(n, c0 + 2000)
        off = wl["pin_off"][c0:c1 + 1] - wl["pin_off"][c0]
        assert g.commit(wf[c0:c1], off, wl["pin_tok"][wl["pin_off"][c0]:wl["pin_off"][c1]]).all()
    Mg, hg = g.match(wf, wl["req_off"], wl["req_tok"], want_hash=True)
    np.testing.assert_array_equal(Mg, wl["expect_M"])
    o = Pool(oracle_api, Config(max_workflows=n, n_blocks=1024, capacity_tokens=1 << 40, max_pin_blocks=mpb,
                                table_log2=12))
    _, ho = o.match(wf, wl["req_off"], wl["req_tok"], want_hash=True)
    np.testing.assert_array_equal(hg, ho)


def test_pool_reserve_grows_in_place(gpu_api, oracle_api):
    """sfkv_pool_reserve: a pool created small grows its workflow slots, block-table length and
    physical blocks (the dedup table re-indexed) mid-stream; every later state equals an oracle
    pool created at the final size (allocation is lowest-free-id, so growth is invisible)."""
    n_wf = 40
    small = Config(max_workflows=8, n_blocks=300, capacity_tokens=60_000, max_pin_blocks=4, table_log2=9)
    big = Config(max_workflows=n_wf, n_blocks=3000, capacity_tokens=60_000, max_pin_blocks=64, table_log2=13)
    g, o = Pool(gpu_api, small), Pool(oracle_api, big)
    wl = Workload(4, n_wf, n_sys=3, sys_len=(16, 60), ctx_len=(0, 40), append=(0, 40))
    rng = np.random.default_rng(4)
    for step in range(10):
        if step == 2:
            gpu_api.check("pool_reserve", gpu_api.pool_reserve(g.h, 16, 16, 900))
        if step == 5:
            gpu_api.check("pool_reserve", gpu_api.pool_reserve(g.h, n_wf, 64, 3000))
            g.cfg = big
        lim = 8 if step < 2 else (16 if step < 5 else n_wf)
        wfs = rng.choice(lim, size=int(rng.integers(1, lim)), replace=False).astype(np.int32)
        seqs, off, tok = wl.batch(wfs)
        if step < 5:  # the small block tables bound the prompt length until the second reserve
            cap = (4 if step < 2 else 16) * 16
            seqs = [s[:cap] for s in seqs]
            off, tok = csr(seqs)
        np.testing.assert_array_equal(g.match(wfs, off, tok), o.match(wfs, off, tok))
        np.testing.assert_array_equal(g.commit(wfs, off, tok), o.commit(wfs, off, tok))
        bg, hg = g.lookup(off, tok)
        bo, ho = o.lookup(off, tok)
        np.testing.assert_array_equal(bg, bo)
        np.testing.assert_array_equal(hg, ho)
    sg, so = g.stats(), o.stats()
    for k in ("occupancy_tokens", "blocks_in_use", "table_live"):
        assert sg[k] == so[k], k
    np.testing.assert_array_equal(g.refcounts(), o.refcounts())
    for w in range(n_wf):
        np.testing.assert_array_equal(g.pin_blocks(w)[0], o.pin_blocks(w)[0])


def test_lookup_one_pass_and_two_pass_agree_with_oracle(gpu_api, oracle_api):
    """Lookup batches of >= 2048 requests take the one-warp-per-request path (lookup_req_kernel:
    running chain sum, TMA double buffer, probe + verify + parent check in one pass); smaller
    batches take the block/chain two-pass path. Both equal sfo_lookup_batch on the same requests:
    shared and private prefixes, partial hits, empty and sub-block requests, requests of up to
    ~300 blocks (many tiles per warp) and the tail tiles that read past the last full 128-B token row."""
    n_wf = 600
    cfg = Config(max_workflows=n_wf, n_blocks=150_000, capacity_tokens=1 << 40, max_pin_blocks=320,
                 table_log2=19)
    g, o = _pair(gpu_api, oracle_api, cfg)
    wl = Workload(21, n_wf, n_sys=6, sys_len=(16, 700), ctx_len=(0, 4000), append=(0, 60))
    wfs = np.arange(n_wf, dtype=np.int32)
    seqs, off, tok = wl.batch(wfs)
    np.testing.assert_array_equal(g.commit(wfs, off, tok), o.commit(wfs, off, tok))
    rng = np.random.default_rng(22)
    reqs = []
    for i in range(3000):
        base = seqs[int(rng.integers(0, n_wf))]
        u = rng.random()
        if u < 0.05:
            q = np.zeros(0, np.uint32)
        elif u < 0.1:
            q = base[: int(rng.integers(1, 16))]
        elif u < 0.3:  # a rewritten token: a miss mid-prefix, hits may resume after it
            q = base.copy()
            if len(q):
                q[int(rng.integers(0, len(q)))] ^= np.uint32(0x77)
        else:
            q = np.concatenate([base[: int(rng.integers(0, len(base) + 1))],
                                rng.integers(1, 1 << 30, size=int(rng.integers(0, 40))).astype(np.uint32)])
        reqs.append(q.astype(np.uint32))
    off2, tok2 = csr(reqs)
    bo, ho = o.lookup(off2, tok2)
    bg, hg = g.lookup(off2, tok2)  # one pass (3000 requests)
    np.testing.assert_array_equal(hg, ho)
    np.testing.assert_array_equal(bg, bo)
    assert (ho > 0).mean() > 0.5
    # the same requests in batches below the one-pass threshold: the two-pass path
    pos = 0
    for c0 in range(0, 3000, 1000):
        sub = reqs[c0:c0 + 1000]
        so, st = csr(sub)
        b2, h2 = g.lookup(so, st)
        nblk = len(b2)
        np.testing.assert_array_equal(h2, ho[c0:c0 + 1000])
        np.testing.assert_array_equal(b2, bo[pos:pos + nblk])
        pos += nblk


@pytest.mark.parametrize("n_wf,lo,hi", [(300, 1200, 1800), (900, 1500, 2400)])
def test_commit_mid_size_batches(gpu_api, oracle_api, n_wf, lo, hi):
    """Commit batches of 28k-150k blocks (the device-wide new-block rank scan takes its
    three-phase path): block tables, refcounts, statuses and the free-block accounting equal the
    oracle's, across a second overlapping batch."""
    rng = np.random.default_rng(n_wf)
    base = rng.integers(1, 1 << 20, size=hi).astype(np.uint32)
    seqs = []
    for i in range(n_wf):
        L = int(rng.integers(lo, hi))
        s = base[:L].copy() if i % 3 else rng.integers(1, 1 << 20, size=L).astype(np.uint32)
        seqs.append(s)
    wfs = np.arange(n_wf, dtype=np.int32)
    nb = sum((len(s) + 15) // 16 for s in seqs) * 2 + 1024
    cfg = Config(max_workflows=n_wf, n_blocks=nb, capacity_tokens=1 << 40, max_pin_blocks=hi // 16 + 8,
                 table_log2=int(np.ceil(np.log2(2 * nb))) + 1)
    g, o = _pair(gpu_api, oracle_api, cfg)
    off, tok = csr(seqs)
    np.testing.assert_array_equal(g.commit(wfs, off, tok), o.commit(wfs, off, tok))
    _assert_same_state(g, o, range(0, n_wf, 7))
    seqs2 = [np.concatenate([s, rng.integers(1, 99, size=int(rng.integers(0, 40))).astype(np.uint32)]) for s in seqs]
    off2, tok2 = csr(seqs2)
    Mg, hg = g.match(wfs, off2, tok2, want_hash=True)
    Mo, ho = o.match(wfs, off2, tok2, want_hash=True)
    np.testing.assert_array_equal(Mg, Mo)
    np.testing.assert_array_equal(hg, ho)
    np.testing.assert_array_equal(g.commit(wfs, off2, tok2), o.commit(wfs, off2, tok2))
    _assert_same_state(g, o, range(0, n_wf, 5))
