"""Cross-process stage handoff over CUDA IPC (PeerLink / sfkv_handoff_recv_batch) on the GPU.

Two ranks (spawned processes, gloo for the metadata) share device 0 here — gpurun gives one GPU,
and CUDA IPC maps a peer process's allocation on the same device exactly as it maps a peer GPU's
(on the 8-GPU box the pull reads travel over NVLink instead). The receiving rank's pins must equal
what the CPU oracle's in-process handoff produces from the same pools: statuses, tokens, and KV
bytes (rows below M copied on share from the receiver's own older pin, the rest pulled from the
sender's blocks)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SHAPES = [(4, 64), (64, 2048)]  # small rows, and the Llama-3-8B block (2 MiB, 32 KiB extents)
SRC_WF, DST_WF = [0, 1, 2], [5, 6, 7]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _contexts(SLABS, ROW):
    rng = np.random.default_rng(11)
    shared = rng.integers(1, 1 << 20, size=40).astype(np.uint32)
    ctx = [np.concatenate([shared, rng.integers(1, 1 << 20, size=n).astype(np.uint32)])
           for n in (0, 37, 90)]
    older = ctx[2][:61]  # the receiver's older pin of workflow 7 (copy-on-share source)
    stg = rng.integers(0, 256, size=sum(len(c) for c in ctx) * SLABS * ROW, dtype=np.uint8)
    stg_old = rng.integers(0, 256, size=len(older) * SLABS * ROW, dtype=np.uint8)
    return ctx, older, stg, stg_old


def _setup(api, rank, SLABS, ROW):
    from paper_2603_13605_b200.abi import Config, Pool, csr
    cfg = Config(max_workflows=8, n_blocks=256, capacity_tokens=100_000, max_pin_blocks=32,
                 table_log2=10, n_slabs=SLABS, slab_row_bytes=ROW)
    pool = Pool(api, cfg)
    ctx, older, stg, stg_old = _contexts(SLABS, ROW)
    if api.kind == "gpu":  # KV staging is device memory for GPU pools
        import torch
        stg, stg_old = torch.from_numpy(stg).cuda(), torch.from_numpy(stg_old).cuda()
    if rank == 0:
        off, tok = csr(ctx)
        kv_off = np.concatenate([[0], np.cumsum([len(c) * SLABS * ROW for c in ctx])[:-1]]).astype(np.int64)
        assert pool.commit(np.array(SRC_WF, np.int32), off, tok, kv_src=stg, kv_src_off=kv_off).all()
    else:
        off, tok = csr([older])
        assert pool.commit(np.array([7], np.int32), off, tok, kv_src=stg_old,
                           kv_src_off=np.zeros(1, np.int64)).all()
    return pool


def _payload(pool, wf):
    from paper_2603_13605_b200 import dist as sfdist
    return sfdist.gather_pin(pool, wf, device="cuda").cpu().numpy().tobytes()


def _worker(rank, port, q, shape):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    try:
        import torch
        import torch.distributed as dist

        import paper_2603_13605_b200 as pkg
        from paper_2603_13605_b200 import dist as sfdist
        torch.cuda.set_device(0)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        pool = _setup(pkg.api(), rank, *shape)
        link = sfdist.PeerLink(pool, device=0)
        res = {}
        if rank == 0:
            res["ack"] = link.send(SRC_WF, dst=1)
        else:
            res["status"] = link.recv(DST_WF, src=0).tolist()
            res["pins"] = [pool.pin_tokens(w).tolist() for w in DST_WF]
            res["payload"] = [_payload(pool, w) for w in DST_WF]
            res["stats"] = pool.stats()
            # a source block outside the peer's KV region is refused before anything moves
            from paper_2603_13605_b200.abi import SfkvError, csr
            off, tok = csr([np.arange(1, 33, dtype=np.uint32)])
            n_src = pool.cfg.n_blocks
            try:
                pool.handoff_recv(link.peers[0], np.array([4], np.int32), off, tok,
                                  np.array([n_src, 0], np.int32))
                res["oob"] = "accepted"
            except SfkvError as e:
                res["oob"] = e.code
            res["stats_after_oob"] = pool.stats()
        dist.barrier()
        link.close()
        dist.destroy_process_group()
        q.put((rank, res, None))
    except Exception:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("shape", SHAPES)
def test_peerlink_pull_handoff_matches_oracle(oracle_api, shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, shape)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        rank, res, err = q.get(timeout=300)
        assert err is None, err
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
    assert out[0]["ack"] == 1
    # the oracle: the same two pools in one process, handoff one pin at a time
    src, dst = _setup(oracle_api, 0, *shape), _setup(oracle_api, 1, *shape)
    want_status = [src.handoff_to(s, dst, d) for s, d in zip(SRC_WF, DST_WF)]
    assert out[1]["status"] == want_status == [1, 1, 1]
    for i, w in enumerate(DST_WF):
        assert out[1]["pins"][i] == dst.pin_tokens(w).tolist()
        assert out[1]["payload"][i] == _payload_oracle(dst, w), f"KV bytes of workflow {w}"
    so = dst.stats()
    for k in ("occupancy_tokens", "blocks_in_use", "table_live"):
        assert out[1]["stats"][k] == so[k], k
    assert out[1]["oob"] == -1  # SFKV_EINVAL
    assert out[1]["stats_after_oob"] == out[1]["stats"]


def _payload_oracle(pool, wf):
    from paper_2603_13605_b200 import dist as sfdist
    return sfdist.gather_pin(pool, wf).numpy().tobytes()
