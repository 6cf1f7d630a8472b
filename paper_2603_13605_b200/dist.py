"""One process per GPU: the multi-rank host logic.

Each rank owns one backend's KV pool (the path shards by backend). Lookup, retain and
evict are rank-local with no collective. The one real exchange is the stage **handoff**: a stage
mapped to another backend ships the workflow's retained context to that backend's rank:

    header (pin length L)  ->  token ids [L] (u32)  ->  KV rows [slab][L][row] (payload pools)

sent point to point with torch.distributed (the portable message path: `send_pin` / `recv_pin`,
which also runs under gloo in the CPU tests). The receiver commits it as its own pin: M =
LCP(its old pin, tokens) rows come from its old pin by copy-on-share inside sfkv_commit_batch, only
rows [M, L) are read from the message.

The B200 path is `PeerLink`: every rank exports its pool's KV region once as a CUDA IPC handle and
maps its peers' regions, so a handoff ships only metadata (tokens + the source pin's block ids)
and the receiver's commit kernel pulls the payload rows straight out of the sender's HBM over
NVLink (sfkv_handoff_recv_batch): one kernel, no gather, no staging buffer, no NCCL payload copy.
Within one process that owns several GPUs, sfkv_handoff does the same transfer.

The second exchange is the **routing step** (`route_step`): every rank computes its pool's M column
for the whole batch of R stage requests (sfkv_match_batch against the workflows' pins on that
backend), one all-gather of R x 8 B per rank assembles the R x C matrix, and every rank runs the
stage mapper (sfmap_cost_batch: cost argmin + in-order reroute) on it, so all ranks agree on the
assignment without another collective.

`max_over_ranks` / `aggregate_rate` implement bench.py's timing rule (max time over ranks, whole-job
units / that time).

Precondition (ABI, include/sfkv.h): token ids are compared as integers, so every rank that
exchanges pins must number token strings the same way — one shared vocabulary (a tokenizer's
fixed ids, or an interner replicated in the same first-occurrence order). Ids from two
independently grown interners are not comparable. `PeerLink` takes a `token_space` label and
refuses to link ranks whose labels differ.
"""
from __future__ import annotations

import numpy as np

from .abi import BLOCK_TOKENS, Pool, csr


def _dist():
    import torch.distributed as dist
    return dist


def gather_pin(pool: Pool, wf: int, device=None):
    """The pin's KV rows as a flat uint8 tensor [slab][L][row] (on `device`)."""
    L = pool.pinned_token_count(wf)
    nbytes = pool.cfg.n_slabs * L * pool.cfg.slab_row_bytes
    return pool.api.gather_payload(pool, wf, nbytes, device)


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
    staging = pool.api.kv_staging(staging, dev)
    st = pool.commit(wfa, off, t, kv_src=staging, kv_src_off=np.zeros(1, dtype=np.int64),
                     m_expected=np.array([M], dtype=np.int64))
    return int(st[0])


def _meta_device(group=None):
    """Metadata tensors live on the GPU for NCCL groups, on the CPU for gloo."""
    import torch
    dist = _dist()
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


class PeerLink:
    """CUDA-IPC links between the ranks' pools (one process per GPU).

    send(wfs, dst) ships the pins' metadata to rank dst and waits for its ack (the blocks must stay
    resident until the receiver has pulled them); recv(wf_dst, src) commits the incoming contexts
    into this rank's pool with the payload pulled from rank src's pool over NVLink."""

    def __init__(self, pool: Pool, device: int, group=None, token_space: str = "default"):
        import ctypes as C

        from .abi import Peer
        dist = _dist()
        self.pool, self.group = pool, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        handles = [None] * self.world
        dist.all_gather_object(handles, (pool.export(), device, token_space), group=group)
        spaces = {sp for _h, _d, sp in handles}
        if len(spaces) != 1:  # ids of different vocabularies would match unrelated text
            raise ValueError(f"PeerLink: ranks use different token-id spaces {sorted(spaces)}")
        self.peers = {}
        for r, (h, _dev, _sp) in enumerate(handles):
            if r != self.rank:
                self.peers[r] = Peer(pool.api, h, device)
        self._C = C

    def close(self):
        for p in self.peers.values():
            p.close()
        self.peers = {}

    def metadata(self, wfs):
        """CSR (tok_off, tok, src_blocks) of the pins of `wfs` in this rank's pool."""
        toks, blks = [], []
        for w in wfs:
            t, b = self.pool.pin_export(int(w))
            toks.append(t)
            blks.append(b)
        off, tok = csr(toks)
        blocks = np.concatenate(blks).astype(np.int32) if blks else np.zeros(0, np.int32)
        return off, tok, blocks

    def send(self, wfs, dst: int):
        import torch
        dist = _dist()
        dev = _meta_device(self.group)
        off, tok, blocks = self.metadata(wfs)
        hdr = torch.tensor([len(wfs), int(off[-1]), len(blocks)], dtype=torch.int64)
        dist.send(hdr.to(dev), dst, group=self.group)
        dist.send(torch.from_numpy(off).to(dev), dst, group=self.group)
        if off[-1]:
            dist.send(torch.from_numpy(tok[: off[-1]].view(np.int32).copy()).to(dev), dst, group=self.group)
            dist.send(torch.from_numpy(blocks).to(dev), dst, group=self.group)
        ack = torch.zeros(1, dtype=torch.int64, device=dev)
        dist.recv(ack, dst, group=self.group)  # the receiver has pulled every block
        return int(ack.item())

    def recv_metadata(self, src: int):
        import torch
        dist = _dist()
        dev = _meta_device(self.group)
        hdr = torch.zeros(3, dtype=torch.int64, device=dev)
        dist.recv(hdr, src, group=self.group)
        n, T, B = (int(x) for x in hdr.cpu())
        off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        dist.recv(off, src, group=self.group)
        tok = torch.zeros(max(T, 1), dtype=torch.int32, device=dev)
        blocks = torch.zeros(max(B, 1), dtype=torch.int32, device=dev)
        if T:
            dist.recv(tok[:T], src, group=self.group)
            dist.recv(blocks[:B], src, group=self.group)
        return (off.cpu().numpy(), tok.cpu().numpy().view(np.uint32), blocks.cpu().numpy())

    def ack(self, src: int, value: int = 1):
        import torch
        _dist().send(torch.tensor([value], dtype=torch.int64, device=_meta_device(self.group)), src,
                     group=self.group)

    def recv(self, wf_dst, src: int):
        """Receive a batch from rank src, pull its payload over NVLink, ack. Returns statuses."""
        off, tok, blocks = self.recv_metadata(src)
        wf_dst = np.ascontiguousarray(wf_dst, dtype=np.int32)
        assert len(wf_dst) == len(off) - 1
        st = self.pool.handoff_recv(self.peers[src], wf_dst, off, tok, blocks)
        self.ack(src)
        return st


def gather_columns(m_col, group=None):
    """SURVEY §8e exchange 2's collective: every rank contributes its pool's M column (int64[R]);
    returns the R x C request-major matrix on m_col's device. NCCL groups gather in place on the
    GPU (all_gather_into_tensor); gloo groups through the host."""
    dist = _dist()
    import torch
    world = dist.get_world_size(group)
    R = m_col.numel()
    mdev = _meta_device(group)
    m_all = torch.empty(world * R, dtype=torch.int64, device=mdev)
    dist.all_gather_into_tensor(m_all, m_col.to(mdev), group=group)
    return m_all.to(m_col.device).view(world, R).t().contiguous()


def route_step(api, pool: Pool, wf, tok_off, tok, P, O, overhead, prefill, decode, qpen, alternates, depth,
               limit: int, device: int = 0, group=None):
    """SURVEY §8e exchange 2: this rank's backend is candidate `rank`; returns (choice[R], cost[R],
    depth[C]) — identical on every rank. The M column, the gathered matrix and the mapper stay on
    the device: sfkv_match_batch_dev, gather_columns, sfmap_cost_batch_dev."""
    import ctypes as C

    import torch
    world = _dist().get_world_size(group)
    R = len(wf)
    wf = np.ascontiguousarray(wf, dtype=np.int32)
    tok_off = np.ascontiguousarray(tok_off, dtype=np.int64)
    par = [np.ascontiguousarray(x, dtype=np.float64) for x in (overhead, prefill, decode, qpen)]
    alt = None if alternates is None else np.ascontiguousarray(alternates, dtype=np.int32)
    P = np.ascontiguousarray(P, dtype=np.int64)
    O = np.ascontiguousarray(O, dtype=np.int64)
    depth = np.ascontiguousarray(depth, dtype=np.uint64).copy()
    dev = torch.device("cuda", device)
    t = lambda x: torch.from_numpy(x).to(dev)  # noqa: E731
    ptr = lambda x: C.c_void_p(x.data_ptr()) if x is not None else None  # noqa: E731
    d_wf, d_off, d_tok = t(wf), t(tok_off), t(np.ascontiguousarray(tok, dtype=np.uint32).view(np.int32))
    m_col = torch.empty(R, dtype=torch.int64, device=dev)
    api.check("match_dev", api.match_batch_dev(pool.h, R, ptr(d_wf), ptr(d_off), ptr(d_tok), int(tok_off[-1]),
                                               ptr(m_col), None))
    api.check("sync", api.pool_sync(pool.h))
    M = gather_columns(m_col, group)  # R x C, request-major
    d = {k: t(v) for k, v in dict(P=P, O=O, oh=par[0], pf=par[1], dc=par[2], qp=par[3],
                                  dp=depth.view(np.int64)).items()}
    d_alt = t(alt) if alt is not None else None
    choice = torch.empty(R, dtype=torch.int32, device=dev)
    cost = torch.empty(R, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    api.check("cost_batch_dev", api.cost_batch_dev(
        device, R, world, ptr(d["P"]), ptr(M), ptr(d["O"]), ptr(d["oh"]), ptr(d["pf"]), ptr(d["dc"]),
        ptr(d["qp"]), ptr(d_alt), ptr(d["dp"]), int(limit), ptr(choice), ptr(cost),
        C.c_void_p(stream.cuda_stream)))
    stream.synchronize()
    return choice.cpu().numpy(), cost.cpu().numpy(), d["dp"].cpu().numpy().view(np.uint64)


def max_over_ranks(x: float, device=None) -> float:
    """bench.py's timing rule: the job takes as long as its slowest rank."""
    import torch
    dist = _dist()
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_meta_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(local_units: float, local_ms: float, device=None) -> float:
    """Whole-job units per second: sum of units over ranks / max time over ranks."""
    import torch
    dist = _dist()
    ms = max_over_ranks(local_ms, device)
    units = float(local_units)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor([units], dtype=torch.float64, device=_meta_device())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        units = float(t.item())
    return units / (ms / 1e3)


def blocks_of(n_tokens: int) -> int:
    return (n_tokens + BLOCK_TOKENS - 1) // BLOCK_TOKENS
