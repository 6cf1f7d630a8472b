"""One process per GPU: the multi-rank host logic.

Each rank owns one backend's KV pool (the path shards by backend). Lookup, retain and
evict are rank-local with no collective. The one real exchange is the stage **handoff**: a stage
mapped to another backend ships the workflow's retained context to that backend's rank:

    header (pin length L)  ->  token ids [L] (u32)  ->  KV rows [slab][L][row] (payload pools)

sent point to point with torch.distributed (NCCL over NVLink between B200 ranks, gloo on CPU). The
receiver commits it as its own pin: M = LCP(its old pin, tokens) rows come from its old pin by
copy-on-share inside sfkv_commit_batch, only rows [M, L) are read from the message. Within one
process that owns several GPUs, sfkv_handoff does the same transfer as a single peer-pull kernel.

`max_over_ranks` / `aggregate_rate` implement bench.py's timing rule (max time over ranks, whole-job
units / that time).
"""
from __future__ import annotations

import numpy as np

from .abi import BLOCK_TOKENS, Pool, csr


def _dist():
    import torch.distributed as dist
    return dist


def gather_pin(pool: Pool, wf: int, device=None):
    """The pin's KV rows as a flat uint8 tensor [slab][L][row] (torch; on `device` for GPU pools)."""
    import torch
    L = pool.pinned_token_count(wf)
    nbytes = pool.cfg.n_slabs * L * pool.cfg.slab_row_bytes
    if pool.api.kind == "oracle":
        buf = np.zeros(max(nbytes, 1), dtype=np.uint8)
        w = np.array([wf], dtype=np.int32)
        off = np.zeros(1, dtype=np.int64)
        pool.api.check("gather", pool.api.gather(pool.h, 1, w.ctypes.data, buf.ctypes.data,
                                                 off.ctypes.data))
        return torch.from_numpy(buf[:nbytes].copy())
    import ctypes as C
    buf = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=device)
    w = torch.tensor([wf], dtype=torch.int32, device=device)
    off = torch.zeros(1, dtype=torch.int64, device=device)
    pool.api.check("gather_dev", pool.api.gather_dev(pool.h, 1, C.c_void_p(w.data_ptr()),
                                                     C.c_void_p(buf.data_ptr()),
                                                     C.c_void_p(off.data_ptr())))
    pool.api.check("pool_sync", pool.api.pool_sync(pool.h))
    return buf[:nbytes]


def send_pin(pool: Pool, wf: int, dst: int, device=None, group=None):
    """Ship workflow `wf`'s retained context to rank `dst`."""
    import torch
    dist = _dist()
    tokens = pool.pin_tokens(wf)
    L = len(tokens)
    dev = device if device is not None else "cpu"
    dist.send(torch.tensor([L], dtype=torch.int64, device=dev), dst, group=group)
    if L:
        dist.send(torch.from_numpy(tokens.view(np.int32).copy()).to(dev), dst, group=group)
        if pool.cfg.n_slabs:
            dist.send(gather_pin(pool, wf, device).to(dev), dst, group=group)
    return L


def recv_pin(pool: Pool, wf: int, src: int, device=None, group=None):
    """Receive a context from rank `src` and commit it as the pin of `wf`. Returns the commit
    status (1 accepted, 0 capacity rejection, as pin_prompt)."""
    import torch
    dist = _dist()
    dev = device if device is not None else "cpu"
    hdr = torch.zeros(1, dtype=torch.int64, device=dev)
    dist.recv(hdr, src, group=group)
    L = int(hdr.item())
    tok = torch.zeros(max(L, 1), dtype=torch.int32, device=dev)
    if L:
        dist.recv(tok, src, group=group)
    tokens = tok[:L].cpu().numpy().view(np.uint32)
    off, t = csr([tokens])
    wfa = np.array([wf], dtype=np.int32)
    if not pool.cfg.n_slabs or L == 0:
        return int(pool.commit(wfa, off, t)[0])
    S, row = pool.cfg.n_slabs, pool.cfg.slab_row_bytes
    payload = torch.zeros(S * L * row, dtype=torch.uint8, device=dev)
    dist.recv(payload, src, group=group)
    M = int(pool.match(wfa, off, t)[0])
    # staging rows [M, L) per slab; rows below M are copied on share from the old pin
    staging = payload.view(S, L, row)[:, M:, :].contiguous().view(-1)
    if pool.api.kind == "oracle":
        staging = staging.cpu().numpy()
        if staging.size == 0:
            staging = np.zeros(16, dtype=np.uint8)
    elif staging.numel() == 0:
        staging = torch.zeros(16, dtype=torch.uint8, device=dev)
    st = pool.commit(wfa, off, t, kv_src=staging, kv_src_off=np.zeros(1, dtype=np.int64),
                     m_expected=np.array([M], dtype=np.int64))
    return int(st[0])


def max_over_ranks(x: float, device=None) -> float:
    """bench.py's timing rule: the job takes as long as its slowest rank."""
    import torch
    dist = _dist()
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(local_units: float, local_ms: float, device=None) -> float:
    """Whole-job units per second: sum of units over ranks / max time over ranks."""
    import torch
    dist = _dist()
    ms = max_over_ranks(local_ms, device)
    units = float(local_units)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor([units], dtype=torch.float64, device=device or "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        units = float(t.item())
    return units / (ms / 1e3)


def blocks_of(n_tokens: int) -> int:
    return (n_tokens + BLOCK_TOKENS - 1) // BLOCK_TOKENS
