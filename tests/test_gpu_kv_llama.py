"""KV payload parity at the benchmarked block shape (Llama-3-8B: 32 layers x K/V = 64 slabs,
8 KV heads x 128 x bf16 = 2 KiB rows, 16-token blocks of 2 MiB).

Every byte-moving path the bench times — commit scatter from staging, copy-on-share of the
boundary block from the old pin, gather, in-process handoff, pool-exhaustion rollback — runs at
this shape against the CPU oracle (oracle/sfkv_oracle.c, write_block_payload and friends) and must
be byte-identical. Extents are (block, slab) runs of up to 16 rows x 2 KiB = 32 KiB, so the copy
kernel's 8-deep unrolled loop (copy.cu warp_copy) carries almost every byte here; pins are
multi-MB (up to ~25 blocks = 50 MiB)."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_13605_b200.abi import Config, Pool, csr
from scenarios import Workload

pytestmark = pytest.mark.gpu

SLABS, ROW = 64, 2048           # Llama-3-8B KV rows (sfkv_pool_config.n_slabs / slab_row_bytes)
TOK_BYTES = SLABS * ROW         # 128 KiB per token


def _cfg(**kw):
    base = dict(max_workflows=8, n_blocks=480, capacity_tokens=1 << 40, max_pin_blocks=48,
                table_log2=12, n_slabs=SLABS, slab_row_bytes=ROW)
    base.update(kw)
    return Config(**base)


def _staging(torch, gen, seqs, M):
    """Random prefill rows [M, P) per request, layout [slab][P - M][row]; (device, host, offsets)."""
    sizes = [SLABS * (len(s) - int(m)) * ROW for s, m in zip(seqs, M)]
    off = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    total = max(int(sum(sizes)), 16)
    dev = torch.randint(0, 256, (total,), dtype=torch.uint8, device="cuda", generator=gen)
    return dev, dev.cpu().numpy(), off


def _gather_all(gpu_api, oracle_api, g, o, n_wf, torch):
    """Every pin's payload, [slab][L][row] per workflow, from both pools."""
    lens = [o.pinned_token_count(w) for w in range(n_wf)]
    assert lens == [g.pinned_token_count(w) for w in range(n_wf)]
    dst_off = np.concatenate([[0], np.cumsum([SLABS * L * ROW for L in lens])[:-1]]).astype(np.int64)
    total = int(sum(SLABS * L * ROW for L in lens)) + 16
    allw = np.arange(n_wf, dtype=np.int32)
    ho = np.zeros(total, dtype=np.uint8)
    oracle_api.check("gather", oracle_api.gather(o.h, n_wf, allw.ctypes.data, ho.ctypes.data,
                                                 dst_off.ctypes.data))
    dg = torch.zeros(total, dtype=torch.uint8, device="cuda")
    dw, doff = torch.from_numpy(allw).cuda(), torch.from_numpy(dst_off).cuda()
    gpu_api.check("gather_dev", gpu_api.gather_dev(g.h, n_wf, C.c_void_p(dw.data_ptr()),
                                                   C.c_void_p(dg.data_ptr()), C.c_void_p(doff.data_ptr())))
    gpu_api.check("pool_sync", gpu_api.pool_sync(g.h))
    return dg.cpu().numpy(), ho, lens, dst_off


def _assert_same_meta(g, o, n_wf):
    sg, so = g.stats(), o.stats()
    for k in ("occupancy_tokens", "capacity_rejections", "blocks_in_use", "table_live"):
        assert sg[k] == so[k], (k, sg[k], so[k])
    np.testing.assert_array_equal(g.refcounts(), o.refcounts())
    for w in range(n_wf):
        np.testing.assert_array_equal(g.pin_blocks(w)[0], o.pin_blocks(w)[0])


def test_llama_shape_scatter_cow_gather(gpu_api, oracle_api):
    """Six stage waves over 8 workflows sharing two system prompts: appends (copy-on-share of the
    non-aligned boundary block), mid-context rewrites and truncations (partial M), cross-workflow
    dedup of shared blocks (no payload written for them), then gather of every pin."""
    torch = pytest.importorskip("torch")
    n_wf = 8
    cfg = _cfg()
    g, o = Pool(gpu_api, cfg), Pool(oracle_api, cfg)
    wl = Workload(21, n_wf, n_sys=2, sys_len=(40, 80), ctx_len=(0, 80), append=(1, 40))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(21)
    rng = np.random.default_rng(21)
    cow_rows = 0
    for step in range(6):
        wfs = np.sort(rng.choice(n_wf, size=int(rng.integers(3, n_wf + 1)), replace=False)).astype(np.int32)
        seqs, off, tok = wl.batch(wfs)
        M = o.match(wfs, off, tok)
        np.testing.assert_array_equal(g.match(wfs, off, tok), M)
        cow_rows += int(sum(int(m) % 16 for m in M))
        dev, host, kv_off = _staging(torch, gen, seqs, M)
        st_o = o.commit(wfs, off, tok, kv_src=host, kv_src_off=kv_off, m_expected=M)
        st_g = g.commit(wfs, off, tok, kv_src=dev, kv_src_off=kv_off, m_expected=M)
        np.testing.assert_array_equal(st_g, st_o)
        _assert_same_meta(g, o, n_wf)
        dg, ho, lens, _ = _gather_all(gpu_api, oracle_api, g, o, n_wf, torch)
        assert max(lens) * TOK_BYTES > (4 << 20), "want multi-MB pins"
        np.testing.assert_array_equal(dg, ho)
    assert cow_rows > 0, "no copy-on-share happened"
    st = g.stats()
    assert st["blocks_in_use"] < sum(-(-g.pinned_token_count(w) // 16) for w in range(n_wf)), \
        "no cross-workflow block sharing happened"


def test_llama_shape_exhaustion_rolls_back_bytes(gpu_api, oracle_api):
    """A batch whose second request exhausts the physical pool fails with SFKV_EPOOL and moves no
    bytes: the first request's would-be blocks are not written, every resident pin's payload is
    unchanged, and the pool keeps working (the retried batch is byte-identical to the oracle)."""
    torch = pytest.importorskip("torch")
    cfg = _cfg(n_blocks=24, max_pin_blocks=16)
    g, o = Pool(gpu_api, cfg), Pool(oracle_api, cfg)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    rng = np.random.default_rng(5)
    first = [rng.integers(1, 1 << 30, size=150).astype(np.uint32)]  # 10 blocks
    off, tok = csr(first)
    dev, host, kv_off = _staging(torch, gen, first, [0])
    for p, s in ((g, dev), (o, host)):
        assert p.commit(np.array([0], np.int32), off, tok, kv_src=s, kv_src_off=kv_off).all()
    before, ho, _, _ = _gather_all(gpu_api, oracle_api, g, o, 8, torch)
    np.testing.assert_array_equal(before, ho)
    # request 0 extends workflow 0 to 170 tokens (2 new blocks, COW of its boundary block),
    # request 1 needs 14 fresh blocks: 16 > the 14 free blocks
    seqs = [np.concatenate([first[0], rng.integers(1, 1 << 30, size=20).astype(np.uint32)]),
            rng.integers(1, 1 << 30, size=14 * 16).astype(np.uint32)]
    off2, tok2 = csr(seqs)
    M = o.match(np.array([0, 1], np.int32), off2, tok2)
    dev2, host2, kv_off2 = _staging(torch, gen, seqs, M)
    for p, s in ((g, dev2), (o, host2)):
        with pytest.raises(Exception) as ei:
            p.commit(np.array([0, 1], np.int32), off2, tok2, kv_src=s, kv_src_off=kv_off2, m_expected=M)
        assert "EPOOL" in str(ei.value) or "-5" in str(ei.value)
    after, ho2, _, _ = _gather_all(gpu_api, oracle_api, g, o, 8, torch)
    np.testing.assert_array_equal(after, before)
    np.testing.assert_array_equal(ho2, ho)
    _assert_same_meta(g, o, 8)
    # a batch that fits still lands byte-identically afterwards
    seqs3 = seqs[:1]
    off3, tok3 = csr(seqs3)
    M3 = o.match(np.array([0], np.int32), off3, tok3)
    dev3, host3, kv_off3 = _staging(torch, gen, seqs3, M3)
    np.testing.assert_array_equal(
        g.commit(np.array([0], np.int32), off3, tok3, kv_src=dev3, kv_src_off=kv_off3, m_expected=M3),
        o.commit(np.array([0], np.int32), off3, tok3, kv_src=host3, kv_src_off=kv_off3, m_expected=M3))
    dg, ho3, _, _ = _gather_all(gpu_api, oracle_api, g, o, 8, torch)
    np.testing.assert_array_equal(dg, ho3)
    _assert_same_meta(g, o, 8)


def test_llama_shape_handoff(gpu_api, oracle_api):
    """In-process stage handoff (sfkv_handoff) of multi-MB pins into a pool that holds an older,
    shorter pin of the destination workflow (rows below M copied on share on the destination side,
    the rest pulled from the source pool's blocks)."""
    torch = pytest.importorskip("torch")
    cfg = _cfg(n_blocks=160, max_pin_blocks=24)
    ga, gb, oa, ob = Pool(gpu_api, cfg), Pool(gpu_api, cfg), Pool(oracle_api, cfg), Pool(oracle_api, cfg)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(9)
    rng = np.random.default_rng(9)
    seqs = [rng.integers(1, 1 << 30, size=n).astype(np.uint32) for n in (300, 133, 16, 1)]
    wfs = np.arange(len(seqs), dtype=np.int32)
    off, tok = csr(seqs)
    dev, host, kv_off = _staging(torch, gen, seqs, [0] * len(seqs))
    assert ga.commit(wfs, off, tok, kv_src=dev, kv_src_off=kv_off).all()
    assert oa.commit(wfs, off, tok, kv_src=host, kv_src_off=kv_off).all()
    older = [seqs[0][:170]]  # destination's older pin of workflow 6: M = 170 (10 COW rows)
    o6, t6 = csr(older)
    d6, h6, k6 = _staging(torch, gen, older, [0])
    assert gb.commit(np.array([6], np.int32), o6, t6, kv_src=d6, kv_src_off=k6).all()
    assert ob.commit(np.array([6], np.int32), o6, t6, kv_src=h6, kv_src_off=k6).all()
    for s, d in ((0, 6), (1, 1), (2, 2), (3, 3)):
        assert ga.handoff_to(s, gb, d) == oa.handoff_to(s, ob, d) == 1
    _assert_same_meta(gb, ob, 8)
    dg, ho, _, _ = _gather_all(gpu_api, oracle_api, gb, ob, 8, torch)
    np.testing.assert_array_equal(dg, ho)
