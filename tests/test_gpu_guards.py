"""Argument and device-side guards of the `_dev` entry points (include/sfkv.h:42, SFKV_EINVAL).

The `_dev` variants take device pointers and do not synchronise, so the host checks only what it
can see (null and misaligned pointers: the kernels use 16-B vector / TMA loads of the token
buffer); a workflow slot read on the device that is out of range is matched as unpinned, moves no
bytes, and sets the pool's sticky error, which the next sfkv_pool_sync reports once."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_13605_b200.abi import Config, Pool, SfkvError, csr

pytestmark = pytest.mark.gpu


def _pool(api, **kw):
    cfg = dict(max_workflows=8, n_blocks=256, capacity_tokens=10_000, max_pin_blocks=16, table_log2=10)
    cfg.update(kw)
    return Pool(api, Config(**cfg))


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _p(t):
    return C.c_void_p(t.data_ptr())


def test_match_dev_out_of_range_slot_reports_once(gpu_api, oracle_api):
    torch = pytest.importorskip("torch")
    g, o = _pool(gpu_api), _pool(oracle_api)
    rng = np.random.default_rng(3)
    seqs = [rng.integers(1, 1000, size=n).astype(np.uint32) for n in (40, 70, 33)]
    off, tok = csr(seqs)
    wf = np.array([0, 1, 2], np.int32)
    for p in (g, o):
        assert p.commit(wf, off, tok).all()
    bad = np.array([0, 99, 2], np.int32)  # slot 99 >= max_workflows
    d_wf, d_off, d_tok = _dev(torch, bad), _dev(torch, off), _dev(torch, tok.view(np.int32))
    d_M = torch.full((3,), -7, dtype=torch.int64, device="cuda")
    gpu_api.check("match_dev", gpu_api.match_batch_dev(g.h, 3, _p(d_wf), _p(d_off), _p(d_tok), int(off[-1]),
                                                      _p(d_M), None))
    with pytest.raises(SfkvError) as e:
        gpu_api.check("pool_sync", gpu_api.pool_sync(g.h))
    assert e.value.code == -1
    gpu_api.check("pool_sync", gpu_api.pool_sync(g.h))  # reported once, then cleared
    M = d_M.cpu().numpy()
    want = o.match(np.array([0, 2], np.int32), *csr([seqs[0], seqs[2]]))
    assert M[0] == want[0] and M[2] == want[1] and M[1] == 0


def test_commit_dev_out_of_range_slot_changes_nothing(gpu_api):
    torch = pytest.importorskip("torch")
    g = _pool(gpu_api)
    seqs = [np.arange(1, 41, dtype=np.uint32), np.arange(5, 30, dtype=np.uint32)]
    off, tok = csr(seqs)
    assert g.commit(np.array([0, 1], np.int32), off, tok).all()
    before = (g.stats(), g.refcounts().copy(), g.pin_tokens(0).copy())
    d_wf = _dev(torch, np.array([3, -1], np.int32))
    d_off, d_tok = _dev(torch, off), _dev(torch, tok.view(np.int32))
    st = torch.zeros(2, dtype=torch.int32, device="cuda")
    gpu_api.check("commit_dev", gpu_api.commit_batch_dev(g.h, 2, _p(d_wf), _p(d_off), _p(d_tok), int(off[-1]),
                                                        None, None, None, _p(st)))
    with pytest.raises(SfkvError) as e:
        gpu_api.check("pool_sync", gpu_api.pool_sync(g.h))
    assert e.value.code == -1
    assert (st.cpu().numpy() == -1).all()
    after = (g.stats(), g.refcounts(), g.pin_tokens(0))
    assert after[0] == before[0]
    assert (after[1] == before[1]).all() and (after[2] == before[2]).all()
    # the pool keeps working after the report
    assert g.commit(np.array([3], np.int32), *csr([seqs[1]])).all()


def test_dev_entry_points_refuse_misaligned_tokens(gpu_api):
    torch = pytest.importorskip("torch")
    g = _pool(gpu_api)
    off, tok = csr([np.arange(1, 41, dtype=np.uint32)])
    d_wf, d_off = _dev(torch, np.array([0], np.int32)), _dev(torch, off)
    buf = torch.zeros(64, dtype=torch.int32, device="cuda")
    unaligned = C.c_void_p(buf.data_ptr() + 4)  # 4-B aligned, not 16-B
    d_M = torch.zeros(1, dtype=torch.int64, device="cuda")
    assert gpu_api.match_batch_dev(g.h, 1, _p(d_wf), _p(d_off), unaligned, 40, _p(d_M), None) == -1
    assert b"16-byte" in gpu_api.lib.sfkv_last_error()
    d_blk = torch.zeros(8, dtype=torch.int32, device="cuda")
    assert gpu_api.lookup_batch_dev(g.h, 1, _p(d_off), unaligned, 40, _p(d_blk), _p(d_M)) == -1
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    assert gpu_api.commit_batch_dev(g.h, 1, _p(d_wf), _p(d_off), unaligned, 40, None, None, None, _p(st)) == -1
    gpu_api.check("pool_sync", gpu_api.pool_sync(g.h))  # nothing was launched


def test_gather_dev_out_of_range_slot_gathers_nothing(gpu_api):
    torch = pytest.importorskip("torch")
    g = _pool(gpu_api, n_slabs=2, slab_row_bytes=16)
    off, tok = csr([np.arange(1, 41, dtype=np.uint32)])
    stg = torch.randint(0, 256, (2 * 40 * 16,), dtype=torch.uint8, device="cuda")
    assert g.commit(np.array([0], np.int32), off, tok, kv_src=stg, kv_src_off=np.zeros(1, np.int64)).all()
    d_wf = _dev(torch, np.array([0, 50], np.int32))
    d_off = _dev(torch, np.array([0, 2 * 40 * 16], np.int64))
    dst = torch.zeros(2 * 2 * 40 * 16, dtype=torch.uint8, device="cuda")
    gpu_api.check("gather_dev", gpu_api.gather_dev(g.h, 2, _p(d_wf), _p(dst), _p(d_off)))
    with pytest.raises(SfkvError):
        gpu_api.check("pool_sync", gpu_api.pool_sync(g.h))
    out = dst.cpu().numpy()
    assert (out[: 2 * 40 * 16] == stg.cpu().numpy()).all()
    assert (out[2 * 40 * 16:] == 0).all()
