"""N > 1 host logic on CPU (world_size 2, gloo): the cross-rank stage handoff protocol and the
max-over-ranks timing rule. Pools are CPU oracle pools here (the same ABI); on B200 ranks the same
code runs over NCCL with libsfkv pools."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist

    import oracle_lib
    from paper_2603_13605_b200 import dist as sfdist
    from paper_2603_13605_b200.abi import Config, Pool, csr
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        api = oracle_lib.load()
        cfg = Config(max_workflows=8, n_blocks=512, capacity_tokens=100_000, max_pin_blocks=64,
                     table_log2=11, n_slabs=3, slab_row_bytes=16)
        pool = Pool(api, cfg)
        rng = np.random.default_rng(42)
        ctx = rng.integers(1, 1 << 20, size=150).astype(np.uint32)
        result = {}
        if rank == 0:
            # backend 0 served stage 1 of workflow 3: pin + KV rows from its prefill
            off, tok = csr([ctx])
            staging = rng.integers(0, 256, size=3 * 150 * 16, dtype=np.uint8)
            assert pool.commit(np.array([3], np.int32), off, tok, kv_src=staging,
                               kv_src_off=np.zeros(1, np.int64))[0] == 1
            result["sent_len"] = sfdist.send_pin(pool, 3, dst=1)
            result["payload"] = sfdist.gather_pin(pool, 3).numpy().tobytes()
        else:
            # backend 1 already holds an older, shorter context of workflow 5 (copy-on-share source)
            older = ctx[:70]
            off, tok = csr([older])
            stg = np.random.default_rng(42)
            rng2 = np.random.default_rng(7)
            staging = rng2.integers(0, 256, size=3 * 70 * 16, dtype=np.uint8)
            pool.commit(np.array([5], np.int32), off, tok, kv_src=staging,
                        kv_src_off=np.zeros(1, np.int64))
            result["status"] = sfdist.recv_pin(pool, 5, src=0)
            result["pin"] = pool.pin_tokens(5).tolist()
            result["payload"] = sfdist.gather_pin(pool, 5).numpy().tobytes()
            result["old_rows"] = staging.reshape(3, 70, 16)
        # timing rule: rank r took (r + 1) ms for 100 units
        result["rate"] = sfdist.aggregate_rate(100, float(rank + 1))
        result["max"] = sfdist.max_over_ranks(float(rank + 1))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, result, None))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


def test_two_rank_handoff_and_timing_rule():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        rank, res, err = q.get(timeout=240)
        assert err is None, err
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
    assert out[0]["sent_len"] == 150
    assert out[1]["status"] == 1
    rng = np.random.default_rng(42)
    ctx_tok = rng.integers(1, 1 << 20, size=150).astype(np.uint32)
    assert out[1]["pin"] == ctx_tok.tolist()
    sent = np.frombuffer(out[0]["payload"], dtype=np.uint8).reshape(3, 150, 16)
    got = np.frombuffer(out[1]["payload"], dtype=np.uint8).reshape(3, 150, 16)
    # rows below M = 70 were copied on share from the receiver's own older pin; the rest came
    # over the wire
    np.testing.assert_array_equal(got[:, :70, :], out[1]["old_rows"])
    np.testing.assert_array_equal(got[:, 70:, :], sent[:, 70:, :])
    for r in (0, 1):
        assert out[r]["max"] == 2.0
        assert out[r]["rate"] == pytest.approx(200 / 2e-3)


def _route_inputs(world):
    """A shared batch of 64 stage requests and, per backend rank, pins holding different prefixes
    of them (so every candidate column of M differs)."""
    rng = np.random.default_rng(9)
    R = 64
    base = [rng.integers(1, 1 << 20, size=int(rng.integers(20, 200))).astype(np.uint32) for _ in range(R)]
    reqs = [np.concatenate([b, rng.integers(1, 1 << 20, size=int(rng.integers(0, 40))).astype(np.uint32)])
            for b in base]
    pins = [[b[: int(len(b) * f)] for b, f in zip(base, rng.random(R))] for _ in range(world)]
    P = np.array([len(x) for x in reqs], np.int64)
    O = rng.integers(0, 64, size=R).astype(np.int64)
    par = [rng.random(world) * 5, rng.random(world) * 0.5, rng.random(world), rng.random(world) * 3]
    alt = np.full((world, world), -1, np.int32)
    for i in range(world):
        alt[i, : world - 1] = [(i + j) % world for j in range(1, world)]
    return reqs, pins, P, O, par, alt


def _route_worker(rank, world, port, q, kind="oracle"):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist

    import oracle_lib
    from paper_2603_13605_b200 import dist as sfdist
    from paper_2603_13605_b200.abi import Config, Pool, csr
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        if kind == "gpu":  # B200 pools (both ranks on device 0 here: gpurun gives one GPU)
            import torch
            torch.cuda.set_device(0)
            import paper_2603_13605_b200 as pkg
            api = pkg.api()
        else:
            api = oracle_lib.load()
        reqs, pins, P, O, par, alt = _route_inputs(world)
        R = len(reqs)
        pool = Pool(api, Config(max_workflows=R, n_blocks=4096, capacity_tokens=1 << 30, max_pin_blocks=32,
                                table_log2=14))
        wf = np.arange(R, dtype=np.int32)
        assert pool.commit(wf, *csr(pins[rank])).all()
        off, tok = csr(reqs)
        route = sfdist.route_step if kind == "gpu" else oracle_lib.route_step_host
        res = route(api, pool, wf, off, tok, P, O, *par, alt, np.zeros(world, np.uint64), limit=20)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res, None))
    except Exception:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


def _route_check(oracle_api, kind):
    from paper_2603_13605_b200.abi import Config, Pool, csr
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_route_worker, args=(r, world, port, q, kind)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, res, err = q.get(timeout=240)
        assert err is None, err
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
    reqs, pins, P, O, par, alt = _route_inputs(world)
    R = len(reqs)
    wf = np.arange(R, dtype=np.int32)
    off, tok = csr(reqs)
    cols = []
    for b in range(world):
        pool = Pool(oracle_api, Config(max_workflows=R, n_blocks=4096, capacity_tokens=1 << 30, max_pin_blocks=32,
                                       table_log2=14))
        pool.commit(wf, *csr(pins[b]))
        cols.append(pool.match(wf, off, tok))
    M = np.ascontiguousarray(np.stack(cols, 1))
    assert (M[:, 0] != M[:, 1]).any()
    choice, cost, depth = np.zeros(R, np.int32), np.zeros(R, np.float64), np.zeros(world, np.uint64)
    oracle_api.check("cost", oracle_api.cost_batch(R, world, P.ctypes.data, M.ctypes.data, O.ctypes.data,
                                                   *[x.ctypes.data for x in par], alt.ctypes.data,
                                                   depth.ctypes.data, 20, choice.ctypes.data, cost.ctypes.data))
    assert depth.max() >= 20  # the queue limit re-routed part of the batch
    for r in range(world):
        np.testing.assert_array_equal(out[r][0], choice)
        np.testing.assert_array_equal(out[r][1], cost)
        np.testing.assert_array_equal(out[r][2], depth)


def test_two_rank_route_step_matches_single_process(oracle_api):
    """SURVEY §8e exchange 2: each rank's M column + one all-gather + the mapper on every rank gives
    the assignment one process computes from the full R x C matrix (and all ranks agree)."""
    _route_check(oracle_api, "oracle")


@pytest.mark.gpu
def test_two_rank_route_step_on_b200_pools(oracle_api):
    """The same exchange with libsfkv pools: sfkv_match_batch_dev per rank, the all-gather, then
    sfmap_cost_batch_dev on every rank; equal to the oracle's single-process assignment."""
    _route_check(oracle_api, "gpu")
