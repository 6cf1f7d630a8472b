"""ctypes binding of the sfkv C ABI (include/sfkv.h) and a numpy-level pool wrapper.

The product binds only ``libsfkv.so``. The signature tables are module-level so that the tests'
checker binding (tests/oracle_lib.py, the CPU oracle's ``sfo_`` restatement of the same entry
points) can reuse them; nothing in this package loads or branches on the oracle.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

BLOCK_TOKENS = 16
FLUSH_ALL = -1

ERRORS = {
    -1: "SFKV_EINVAL",
    -2: "SFKV_ENODEV",
    -3: "SFKV_ECUDA",
    -4: "SFKV_ENOMEM",
    -5: "SFKV_EPOOL",
    -6: "SFKV_ESTALE",
}


class PoolConfig(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("max_workflows", C.c_int32),
        ("n_blocks", C.c_int64),
        ("capacity_tokens", C.c_int64),
        ("max_pin_blocks", C.c_int32),
        ("table_log2", C.c_int32),
        ("n_slabs", C.c_int32),
        ("slab_row_bytes", C.c_int32),
    ]


class IpcHandle(C.Structure):  # sfkv_ipc_handle
    _fields_ = [
        ("handle", C.c_char * 64),
        ("kv_bytes", C.c_int64),
        ("block_bytes", C.c_int64),
        ("n_slabs", C.c_int32),
        ("slab_row_bytes", C.c_int32),
    ]


class PoolStats(C.Structure):
    _fields_ = [
        ("occupancy_tokens", C.c_int64),
        ("capacity_tokens", C.c_int64),
        ("capacity_rejections", C.c_uint64),
        ("flush_calls", C.c_uint64),
        ("preserve_calls", C.c_uint64),
        ("blocks_in_use", C.c_int64),
        ("table_live", C.c_int64),
        ("table_tombstones", C.c_int64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


P = C.c_void_p
i32, i64, u32, u64, f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double

# name -> argtypes (all return int unless listed in _RESTYPES)
SIGNATURES = {
    "pool_create": [C.POINTER(PoolConfig), C.POINTER(P)],
    "pool_destroy": [P],
    "pool_kv": [P, C.POINTER(P), C.POINTER(i64)],
    "match_batch": [P, i64, P, P, P, P, P],
    "lookup_batch": [P, i64, P, P, P, P],
    "commit_batch": [P, i64, P, P, P, P, P, P, P],
    "flush": [P, i32, C.POINTER(i64)],
    "flush_batch": [P, i64, P, P],
    "preserve": [P, i32, C.POINTER(i32)],
    "pinned_token_count": [P, i32, C.POINTER(i64)],
    "cache_utilization": [P, C.POINTER(f64)],
    "stats": [P, C.POINTER(PoolStats)],
    "pin_blocks": [P, i32, P, P, i32, C.POINTER(i32)],
    "block_refcounts": [P, P],
    "pin_tokens": [P, i32, P, i64, C.POINTER(i64)],
    "handoff": [P, i32, P, i32, C.POINTER(i32)],
    "block_digest": [u64, u32, P],
    "interner_create": [i32, i32, i64, C.POINTER(P)],
    "interner_destroy": [P],
    "interner_size": [P, C.POINTER(i64)],
    "interner_token": [P, u32, P, i32, C.POINTER(i32)],
    "tokenize_batch": [P, i64, P, P, P, P, P, i64, C.POINTER(i64)],
    "chain_finalize": [u64],
}
# entry points without a counterpart in SIGNATURES' shared list
GPU_ONLY = {
    "abi_version": [],
    "last_error": [],
    "pool_set_stream": [P, P],
    "pool_reserve": [P, i32, i32, i64],
    "pool_config_get": [P, C.POINTER(PoolConfig)],
    "pool_sync": [P],
    "match_batch_dev": [P, i64, P, P, P, i64, P, P],
    "lookup_batch_dev": [P, i64, P, P, i64, P, P],
    "commit_batch_dev": [P, i64, P, P, P, i64, P, P, P, P],
    "gather_dev": [P, i64, P, P, P],
    "interner_set_stream": [P, P],
    "interner_check": [P],
    "interner_reserve": [P, i32, i64],
    "interner_arena": [P, C.POINTER(i64), C.POINTER(i64), C.POINTER(i32)],
    "interner_reset": [P],
    "tokenize_batch_dev": [P, i64, P, i64, P, P, i64, P, P, P],
    "pool_export": [P, C.POINTER(IpcHandle)],
    "peer_open": [C.POINTER(IpcHandle), i32, C.POINTER(P)],
    "peer_close": [P],
    "pin_export": [P, i32, P, P, i64, C.POINTER(i64)],
    "handoff_recv_batch": [P, P, i64, P, P, P, P, P],
    "handoff_recv_batch_dev": [P, P, i64, P, P, P, i64, P, P],
}
MET_FNS = {  # sfmet_* (first argument: device ordinal)
    "latency_batch": [P, i64, P, P, P, P, P, i32, P, P, P, P, P, P],
    "nearest_rank": [P, i64, P, i32, P, P],
}
GLOBAL_FNS = {  # sfmm_pressure_argmin / sfmap_* (first argument: device ordinal)
    "pressure_argmin": [P, i64, P, P, P, P, P, i32, P, f64, P],
    "threshold_batch": [P, i64, P, f64, P],
    "cost_batch": [P, i64, i32, P, P, P, P, P, P, P, P, P, u64, P, P],
}
# memory-manager tracker: sfmm_*
MM_FNS = {
    "tracker_create": [P, C.POINTER(P)],
    "tracker_destroy": [P],
    "set_workflow_chain": [P, i32, i32, P],
    "set_workflow_ranks": [P, i64, P],
    "on_signal_batch": [P, i64, P, P],
    "pressure_tick": [P, P, P],
    "tracker_entries": [P, P, P, P, P, P],
    "tracker_reserve": [P, i32, i32, i32],
    "tracker_shape": [P, P, P, P],
    "reset_workflows": [P, i64, P],
    "set_backend_order": [P, i32, P],
    "flush_failed": [P, i64, P, P, P],
}
MM_GPU_ONLY = {
    "tracker_set_stream": [P, P],
    "tracker_sync": [P],
    "tracker_reset": [P],
    "on_signal_batch_dev": [P, i64, P, P],
    "pressure_tick_dev": [P, P, P],
}
_RESTYPES = {
    "block_digest": u64,
    "chain_finalize": u64,
    "last_error": C.c_char_p,
    "chain_hashes": None,
}


class SfkvError(RuntimeError):
    def __init__(self, fn, code, detail=""):
        super().__init__(f"{fn} failed: {ERRORS.get(code, code)} {detail}".strip())
        self.code = code


class Api:
    """Bound entry points of libsfkv.so: ``api.match_batch(...)`` etc. (raw ints returned).

    The product binds nothing else. Calls whose argument lists carry a device ordinal go through
    ``dev_call``; the few pool operations that move payload bytes between a pool and torch
    (``gather_payload`` / ``kv_staging``) are methods here so that code above the binding stays
    free of per-library branches."""

    kind = "gpu"

    def __init__(self, lib: C.CDLL):
        self.lib = lib
        self._bind_tables()

    def _bind_tables(self):
        table = dict(SIGNATURES)
        table.update(GPU_ONLY)
        for name, argt in table.items():
            self._bind("sfkv_" + name, name, argt)
        for name, argt in {**MM_FNS, **MM_GPU_ONLY}.items():
            self._bind("sfmm_" + name, "mm_" + name, argt)
        for name, argt in MET_FNS.items():
            self._bind("sfmet_" + name, name, [i32] + argt[1:])
        for name, argt in GLOBAL_FNS.items():
            sym = ("sfmm_" if name == "pressure_argmin" else "sfmap_") + name
            self._bind(sym, name, [i32] + argt[1:])  # first arg: device ordinal
        # device-pointer mapper batch (+ stream)
        self._bind("sfmap_cost_batch_dev", "cost_batch_dev", [i32] + GLOBAL_FNS["cost_batch"][1:] + [P])

    def _bind(self, sym, name, argt):
        fn = getattr(self.lib, sym)
        fn.argtypes = argt
        fn.restype = _RESTYPES.get(name, C.c_int)
        setattr(self, name, fn)

    def dev_call(self, name: str, device: int, *args):
        """Entry points of MET_FNS / GLOBAL_FNS: the device ordinal leads the argument list."""
        return getattr(self, name)(int(device), *args)

    def error_detail(self) -> str:
        msg = self.lib.sfkv_last_error()
        return msg.decode() if msg else ""

    def check(self, fn: str, rc: int):
        if rc != 0:
            raise SfkvError(fn, rc, self.error_detail())

    # -- payload movement between a pool and torch (device memory) ------------------------------
    def gather_payload(self, pool: "Pool", wf: int, nbytes: int, device=None):
        """The pin's KV rows [slab][L][row] as a flat uint8 device tensor (sfkv_gather_dev)."""
        import torch
        buf = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=device)
        w = torch.tensor([wf], dtype=torch.int32, device=device)
        off = torch.zeros(1, dtype=torch.int64, device=device)
        self.check("gather_dev", self.gather_dev(pool.h, 1, C.c_void_p(w.data_ptr()),
                                                 C.c_void_p(buf.data_ptr()), C.c_void_p(off.data_ptr())))
        self.check("pool_sync", self.pool_sync(pool.h))
        return buf[:nbytes]

    def kv_staging(self, staging, device=None):
        """A commit's kv_src argument from a torch byte tensor: device memory, never empty."""
        import torch
        if staging.numel() == 0:
            return torch.zeros(16, dtype=torch.uint8, device=device)
        return staging


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data_as(C.c_void_p)
    if hasattr(a, "data_ptr"):  # torch tensor (device pointer for *_dev entry points)
        return C.c_void_p(a.data_ptr())
    return a


def csr(seqs):
    """List of token sequences -> (tok_off int64[n+1], tok uint32[total])."""
    off = np.zeros(len(seqs) + 1, dtype=np.int64)
    for i, s in enumerate(seqs):
        off[i + 1] = off[i] + len(s)
    tok = np.zeros(max(int(off[-1]), 1), dtype=np.uint32)
    for i, s in enumerate(seqs):
        tok[off[i]:off[i + 1]] = np.asarray(s, dtype=np.uint32)
    return off, tok


def n_blocks_of(tok_off):
    lens = np.diff(tok_off)
    return (lens + BLOCK_TOKENS - 1) // BLOCK_TOKENS


@dataclass
class Config:
    max_workflows: int = 64
    n_blocks: int = 4096
    capacity_tokens: int = 1_000_000
    max_pin_blocks: int = 256
    table_log2: int = 14
    n_slabs: int = 0
    slab_row_bytes: int = 0
    device: int = 0

    def c(self):
        return PoolConfig(self.device, self.max_workflows, self.n_blocks, self.capacity_tokens,
                          self.max_pin_blocks, self.table_log2, self.n_slabs, self.slab_row_bytes)

    @property
    def block_bytes(self):
        return self.n_slabs * BLOCK_TOKENS * self.slab_row_bytes


class Pool:
    """numpy-level wrapper over one pool handle (host-pointer entry points)."""

    def __init__(self, api: Api, cfg: Config):
        self.api, self.cfg = api, cfg
        h = C.c_void_p()
        api.check("pool_create", api.pool_create(C.byref(cfg.c()), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.api.pool_destroy(self.h)
            self.h = None

    def reserve(self, max_workflows=0, max_pin_blocks=0, n_blocks=0):
        """Grow the pool in place (sfkv_pool_reserve); never shrinks. Updates cfg."""
        mw = max(int(max_workflows), self.cfg.max_workflows)
        mb = max(int(max_pin_blocks), self.cfg.max_pin_blocks)
        nb = max(int(n_blocks), self.cfg.n_blocks)
        self.api.check("pool_reserve", self.api.pool_reserve(self.h, mw, mb, nb))
        c = PoolConfig()
        self.api.check("pool_config_get", self.api.pool_config_get(self.h, C.byref(c)))
        self.cfg.max_workflows, self.cfg.max_pin_blocks = c.max_workflows, c.max_pin_blocks
        self.cfg.n_blocks, self.cfg.table_log2 = c.n_blocks, c.table_log2

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- lookup ---------------------------------------------------------------------------
    def match(self, wf, tok_off, tok, want_hash=False):
        wf = np.ascontiguousarray(wf, dtype=np.int32)
        M = np.zeros(len(wf), dtype=np.int64)
        h = np.zeros(max(int(n_blocks_of(tok_off).sum()), 1), dtype=np.uint64) if want_hash else None
        self.api.check("match_batch", self.api.match_batch(self.h, len(wf), _ptr(wf), _ptr(tok_off),
                                                           _ptr(tok), _ptr(M), _ptr(h)))
        return (M, h[: int(n_blocks_of(tok_off).sum())]) if want_hash else M

    def lookup(self, tok_off, tok):
        n = len(tok_off) - 1
        nfull = int(n_blocks_of(tok_off).sum())
        out = np.zeros(max(nfull, 1), dtype=np.int32)
        hit = np.zeros(n, dtype=np.int64)
        self.api.check("lookup_batch", self.api.lookup_batch(self.h, n, _ptr(tok_off), _ptr(tok),
                                                             _ptr(out), _ptr(hit)))
        return out[:nfull], hit

    # -- retain / evict -------------------------------------------------------------------
    def commit(self, wf, tok_off, tok, kv_src=None, kv_src_off=None, m_expected=None):
        wf = np.ascontiguousarray(wf, dtype=np.int32)
        st = np.zeros(len(wf), dtype=np.int32)
        self.api.check("commit_batch", self.api.commit_batch(
            self.h, len(wf), _ptr(wf), _ptr(tok_off), _ptr(tok), _ptr(kv_src), _ptr(kv_src_off),
            _ptr(m_expected), _ptr(st)))
        return st

    def flush(self, wf):
        out = C.c_int64()
        self.api.check("flush", self.api.flush(self.h, int(wf), C.byref(out)))
        return out.value

    def flush_batch(self, wf):
        wf = np.ascontiguousarray(wf, dtype=np.int32)
        out = np.zeros(len(wf), dtype=np.int64)
        self.api.check("flush_batch", self.api.flush_batch(self.h, len(wf), _ptr(wf), _ptr(out)))
        return out

    def preserve(self, wf):
        out = C.c_int32()
        self.api.check("preserve", self.api.preserve(self.h, int(wf), C.byref(out)))
        return bool(out.value)

    def pinned_token_count(self, wf):
        out = C.c_int64()
        self.api.check("pinned_token_count", self.api.pinned_token_count(self.h, int(wf), C.byref(out)))
        return out.value

    def cache_utilization(self):
        out = C.c_double()
        self.api.check("cache_utilization", self.api.cache_utilization(self.h, C.byref(out)))
        return out.value

    def stats(self):
        s = PoolStats()
        self.api.check("stats", self.api.stats(self.h, C.byref(s)))
        return s.as_dict()

    def pin_blocks(self, wf):
        cap = self.cfg.max_pin_blocks
        ids = np.zeros(cap, dtype=np.int32)
        hs = np.zeros(cap, dtype=np.uint64)
        n = C.c_int32()
        self.api.check("pin_blocks", self.api.pin_blocks(self.h, int(wf), _ptr(ids), _ptr(hs), cap,
                                                         C.byref(n)))
        return ids[: n.value], hs[: n.value]

    def refcounts(self):
        out = np.zeros(self.cfg.n_blocks, dtype=np.uint32)
        self.api.check("block_refcounts", self.api.block_refcounts(self.h, _ptr(out)))
        return out

    def pin_tokens(self, wf):
        n = C.c_int64()
        self.api.check("pin_tokens", self.api.pin_tokens(self.h, int(wf), None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), dtype=np.uint32)
        self.api.check("pin_tokens", self.api.pin_tokens(self.h, int(wf), _ptr(out), n.value,
                                                         C.byref(n)))
        return out[: n.value]

    def handoff_to(self, wf_src, dst: "Pool", wf_dst):
        st = C.c_int32()
        self.api.check("handoff", self.api.handoff(self.h, int(wf_src), dst.h, int(wf_dst),
                                                   C.byref(st)))
        return st.value

    # -- cross-process handoff (GPU pools only) ----------------------------------------------
    def export(self) -> bytes:
        """The pool's KV region as a CUDA IPC handle (sfkv_ipc_handle bytes)."""
        h = IpcHandle()
        self.api.check("pool_export", self.api.pool_export(self.h, C.byref(h)))
        return bytes(C.string_at(C.addressof(h), C.sizeof(h)))

    def pin_export(self, wf):
        """(tokens uint32[L], block ids int32[ceil(L/16)]) of workflow wf's pin."""
        n = C.c_int64()
        self.api.check("pin_export", self.api.pin_export(self.h, int(wf), None, None, 0, C.byref(n)))
        L = n.value
        tok = np.zeros(max(L, 1), dtype=np.uint32)
        ids = np.zeros(max((L + BLOCK_TOKENS - 1) // BLOCK_TOKENS, 1), dtype=np.int32)
        self.api.check("pin_export", self.api.pin_export(self.h, int(wf), _ptr(tok), _ptr(ids), L,
                                                         C.byref(n)))
        return tok[:L], ids[: (L + BLOCK_TOKENS - 1) // BLOCK_TOKENS]

    def handoff_recv(self, peer: "Peer", wf, tok_off, tok, src_blocks):
        """Commit a batch of contexts whose payload is pulled from `peer`'s blocks."""
        wf = np.ascontiguousarray(wf, dtype=np.int32)
        st = np.zeros(len(wf), dtype=np.int32)
        src_blocks = np.ascontiguousarray(src_blocks, dtype=np.int32)
        self.api.check("handoff_recv_batch", self.api.handoff_recv_batch(
            self.h, peer.h, len(wf), _ptr(wf), _ptr(tok_off), _ptr(tok), _ptr(src_blocks), _ptr(st)))
        return st

    def kv_ptr(self):
        p, bb = C.c_void_p(), C.c_int64()
        self.api.check("pool_kv", self.api.pool_kv(self.h, C.byref(p), C.byref(bb)))
        return p.value, bb.value


class Peer:
    """Another process's pool payload mapped into this one (sfkv_peer_open over CUDA IPC)."""

    def __init__(self, api: Api, handle: bytes, device: int):
        h = IpcHandle.from_buffer_copy(handle)
        self.api = api
        self.h = C.c_void_p()
        api.check("peer_open", api.peer_open(C.byref(h), int(device), C.byref(self.h)))

    def close(self):
        if self.h:
            self.api.peer_close(self.h)
            self.h = None


# ---------------------------------------------------------------- memory-manager tracker ----
MM_START, MM_COMPLETE, MM_WF_COMPLETE = 0, 1, 2
MM_OVERRIDE = {"none": 0, "preserve": 1, "flush": 2}
MM_POLICY = {"preserve_small_increment": 1, "flush_at_boundary": 2}
MM_ACT = ["preserve", "flush", "noop"]
MM_REASON = ["override", "preserve_small_increment", "flush_at_boundary", "flush_under_pressure",
             "chain_exhausted"]


class MmConfig(C.Structure):  # sfmm_config / sfo_mm_config
    _fields_ = [
        ("device", C.c_int32),
        ("max_workflows", C.c_int32),
        ("n_backends", C.c_int32),
        ("max_stages", C.c_int32),
        ("chain_len", C.c_int32),
        ("chain", C.c_void_p),
        ("tau", C.c_int64),
        ("tau_pressure", C.c_double),
    ]


class MmSignals(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in
                ("kind", "wf", "stage", "backend", "model", "tokens", "ts", "override_")]


class MmRecords(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in ("count", "status", "kind", "backend", "reason")]


class Tracker:
    """GPU-resident MemoryManager tracker over dense ids (host-pointer entry points)."""

    def __init__(self, api: Api, max_workflows: int, n_backends: int, chain=("preserve_small_increment",
                 "flush_at_boundary"), tau=512, tau_pressure=0.85, device=0, max_stages=0):
        cfg = MmConfig()
        cfg.device, cfg.max_workflows, cfg.n_backends = device, max_workflows, n_backends
        cfg.max_stages = max_stages
        codes = np.array([MM_POLICY[c] for c in chain] or [0], dtype=np.uint8)
        cfg.chain_len, cfg.chain = len(chain), codes.ctypes.data
        cfg.tau, cfg.tau_pressure = tau, tau_pressure
        self.api, self.W, self.NB = api, max_workflows, n_backends
        self.h = C.c_void_p()
        api.check("tracker_create", api.mm_tracker_create(C.byref(cfg), C.byref(self.h)))

    def reserve(self, max_workflows=0, n_backends=0, max_stages=0):
        self.api.check("tracker_reserve", self.api.mm_tracker_reserve(self.h, max_workflows, n_backends, max_stages))
        w, b, s = C.c_int32(), C.c_int32(), C.c_int32()
        self.api.check("tracker_shape", self.api.mm_tracker_shape(self.h, C.byref(w), C.byref(b), C.byref(s)))
        self.W, self.NB = w.value, b.value
        return w.value, b.value, s.value

    def reset_workflows(self, wf):
        wf = np.ascontiguousarray(wf, np.int32)
        self.api.check("reset_workflows", self.api.mm_reset_workflows(self.h, len(wf), _ptr(wf)))

    def set_backend_order(self, order):
        order = np.ascontiguousarray(order, np.int32)
        self.api.check("set_backend_order", self.api.mm_set_backend_order(self.h, len(order), _ptr(order)))

    def flush_failed(self, wf, backend, sig):
        """Flush records that failed twice (sig = index in the last batch, -1 = the last tick)."""
        wf, backend = np.ascontiguousarray(wf, np.int32), np.ascontiguousarray(backend, np.int32)
        sig = np.ascontiguousarray(sig, np.int64)
        self.api.check("flush_failed", self.api.mm_flush_failed(self.h, len(wf), _ptr(wf), _ptr(backend), _ptr(sig)))

    def close(self):
        if self.h:
            self.api.mm_tracker_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_chain(self, wf, names):
        codes = np.array([MM_POLICY[n] for n in names] or [0], dtype=np.uint8)
        self.api.check("set_workflow_chain", self.api.mm_set_workflow_chain(
            self.h, int(wf), len(names), _ptr(codes)))

    def set_ranks(self, rank):
        rank = np.ascontiguousarray(rank, dtype=np.uint32)
        self.api.check("set_workflow_ranks", self.api.mm_set_workflow_ranks(self.h, len(rank), _ptr(rank)))

    def on_signals(self, kind, wf, stage, backend, model, tokens, ts, override):
        """Arrays of n signals -> (count[n], status[n], kind[n,NB], backend[n,NB], reason[n,NB])."""
        n = len(kind)
        arrs = [np.ascontiguousarray(kind, np.uint8), np.ascontiguousarray(wf, np.int32),
                np.ascontiguousarray(stage, np.int32), np.ascontiguousarray(backend, np.int32),
                np.ascontiguousarray(model, np.int32), np.ascontiguousarray(tokens, np.int64),
                np.ascontiguousarray(ts, np.float64), np.ascontiguousarray(override, np.uint8)]
        sig = MmSignals(*[a.ctypes.data for a in arrs])
        cnt = np.zeros(n, np.int32)
        st = np.zeros(n, np.uint8)
        k = np.zeros(max(n * self.NB, 1), np.uint8)
        b = np.zeros(max(n * self.NB, 1), np.int32)
        r = np.zeros(max(n * self.NB, 1), np.uint8)
        rec = MmRecords(cnt.ctypes.data, st.ctypes.data, k.ctypes.data, b.ctypes.data, r.ctypes.data)
        self.api.check("on_signal_batch", self.api.mm_on_signal_batch(self.h, n, C.byref(sig), C.byref(rec)))
        nb = self.NB
        return cnt, st, k[: n * nb].reshape(n, nb), b[: n * nb].reshape(n, nb), r[: n * nb].reshape(n, nb)

    def pressure_tick(self, util):
        util = np.ascontiguousarray(util, np.float64)
        out = np.zeros(self.NB, np.int32)
        self.api.check("pressure_tick", self.api.mm_pressure_tick(self.h, _ptr(util), _ptr(out)))
        return out

    def entries(self):
        E = self.W * self.NB
        pres, keep = np.zeros(E, np.uint8), np.zeros(E, np.uint8)
        tok, ts, inf = np.zeros(E, np.int64), np.zeros(E, np.float64), np.zeros(E, np.int32)
        self.api.check("tracker_entries", self.api.mm_tracker_entries(
            self.h, _ptr(pres), _ptr(keep), _ptr(tok), _ptr(ts), _ptr(inf)))
        shp = (self.W, self.NB)
        return (pres.reshape(shp), keep.reshape(shp), tok.reshape(shp), ts.reshape(shp), inf.reshape(shp))


# ---------------------------------------------------------------- tokenizer + interner ------
def text_batch(requests):
    """requests: list of lists of message byte strings -> (req_msg_off, msg_off, text u8)."""
    req = np.zeros(len(requests) + 1, np.int64)
    msgs = []
    for i, r in enumerate(requests):
        req[i + 1] = req[i] + len(r)
        msgs.extend(r)
    moff = np.zeros(len(msgs) + 1, np.int64)
    for i, m in enumerate(msgs):
        moff[i + 1] = moff[i] + len(m)
    text = np.frombuffer(b"".join(msgs) + b"\0" * 16, dtype=np.uint8).copy()
    return req, moff, text


class Interner:
    """Token-string interner + whitespace tokenizer (host-pointer entry points)."""

    def __init__(self, api: Api, table_log2=20, arena_bytes=64 << 20, device=0):
        self.api = api
        self.h = C.c_void_p()
        api.check("interner_create", api.interner_create(device, table_log2, arena_bytes, C.byref(self.h)))

    def close(self):
        if self.h:
            self.api.interner_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def arena(self):
        """(arena bytes used, arena capacity, table log2)."""
        u, c, lg = C.c_int64(), C.c_int64(), C.c_int32()
        self.api.check("interner_arena", self.api.interner_arena(self.h, C.byref(u), C.byref(c), C.byref(lg)))
        return u.value, c.value, lg.value

    def reset(self):
        """Forget every string (sfkv_interner_reset); allocations and batch scratch are kept."""
        self.api.check("interner_reset", self.api.interner_reset(self.h))

    def reserve(self, table_log2, arena_bytes):
        """Grow in place (sfkv_interner_reserve); every existing string keeps its id."""
        self.api.check("interner_reserve", self.api.interner_reserve(self.h, int(table_log2), int(arena_bytes)))

    def tokenize_growing(self, requests, max_grow=16):
        """tokenize(); on a full table / arena (SFKV_EPOOL: the batch changed nothing) reserve twice
        the size and retry."""
        for attempt in range(max_grow + 1):
            try:
                return self.tokenize(requests)
            except SfkvError as e:
                if e.code != -5 or attempt == max_grow:
                    raise
                used, cap, lg = self.arena()
                nbytes = sum(len(m) for r in requests for m in r)
                self.reserve(lg + 1, max(2 * cap, used + 2 * nbytes + 4096))

    def tokenize(self, requests):
        """-> (tok_off int64[n+1], tok uint32[T]) for a list of requests (lists of messages)."""
        req, moff, text = text_batch(requests)
        nbytes = int(moff[-1])
        cap = max((nbytes + len(moff) - 1 + 1) // 2, 1)  # (n_bytes + n_msg + 1) / 2
        tok_off = np.zeros(len(requests) + 1, np.int64)
        tok = np.zeros(cap, np.uint32)
        nt = C.c_int64()
        self.api.check("tokenize_batch", self.api.tokenize_batch(
            self.h, len(requests), _ptr(req), _ptr(moff), _ptr(text), _ptr(tok_off), _ptr(tok), cap,
            C.byref(nt)))
        return tok_off, tok[: nt.value]

    def size(self):
        n = C.c_int64()
        self.api.check("interner_size", self.api.interner_size(self.h, C.byref(n)))
        return n.value

    def token(self, i):
        ln = C.c_int32()
        self.api.check("interner_token", self.api.interner_token(self.h, int(i), None, 0, C.byref(ln)))
        buf = C.create_string_buffer(max(ln.value, 1))
        self.api.check("interner_token", self.api.interner_token(self.h, int(i), buf, ln.value, C.byref(ln)))
        return buf.raw[: ln.value]


# ---------------------------------------------------------------- latency model / metrics ---
def latency_batch(api: Api, backend, queue_ms, P, M, O, overhead, prefill, decode, device=0):
    """(ttft, total, service) per request: SimulatedBackend::start's timing, batched."""
    n = len(backend)
    arrs = [np.ascontiguousarray(backend, np.int32), np.ascontiguousarray(queue_ms, np.float64),
            np.ascontiguousarray(P, np.int64), np.ascontiguousarray(M, np.int64), np.ascontiguousarray(O, np.int64)]
    par = [np.ascontiguousarray(x, np.float64) for x in (overhead, prefill, decode)]
    ttft, total, svc = np.zeros(n), np.zeros(n), np.zeros(n)
    args = [n] + [_ptr(a) for a in arrs] + [len(par[0])] + [_ptr(x) for x in par] + [_ptr(ttft), _ptr(total), _ptr(svc)]
    api.check("latency_batch", api.dev_call("latency_batch", device, *args))
    return ttft, total, svc


def nearest_rank(api: Api, samples, pct, device=0):
    samples = np.ascontiguousarray(samples, np.float64)
    pct = np.ascontiguousarray(pct, np.int32)
    out = np.zeros(len(pct))
    args = [len(samples), _ptr(samples), len(pct), _ptr(pct), _ptr(out)]
    api.check("nearest_rank", api.dev_call("nearest_rank", device, *args))
    return out
