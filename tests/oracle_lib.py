"""Loads the CPU oracle (oracle/_build/libsfkv_oracle.so) and the reference shim
(oracle/_ref/libsfref.so). Test infrastructure only: the checker, never the thing measured.

``OracleApi`` binds the oracle's ``sfo_`` restatement of include/sfkv.h under the same attribute
names as the product binding (paper_2603_13605_b200.abi.Api), so a test drives both libraries with
identical arguments. The product package knows nothing about this class."""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2603_13605_b200.abi import (GLOBAL_FNS, MET_FNS, MM_FNS, SIGNATURES, Api, P, SfkvError,
                                       i64)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(REPO, "oracle", "_build", "libsfkv_oracle.so")
REF_SO = os.path.join(REPO, "oracle", "_ref", "libsfref.so")
_cache = {}

ORACLE_ONLY = {
    "gather": [P, i64, P, P, P],
    "chain_hashes": [P, i64, P],
}


class OracleApi(Api):
    """The oracle's entry points: host pointers everywhere, no device ordinal."""

    kind = "oracle"

    def _bind_tables(self):
        table = dict(SIGNATURES)
        table.update(ORACLE_ONLY)
        for name, argt in table.items():
            self._bind("sfo_" + name, name, argt)
        for name, argt in MM_FNS.items():
            self._bind("sfo_" + name, "mm_" + name, argt)
        for name, argt in {**MET_FNS, **GLOBAL_FNS}.items():
            self._bind("sfo_" + name, name, argt[1:])

    def dev_call(self, name, device, *args):
        return getattr(self, name)(*args)

    def error_detail(self):
        return ""

    def check(self, fn, rc):
        if rc != 0:
            raise SfkvError(fn, rc)

    def gather_payload(self, pool, wf, nbytes, device=None):
        import torch
        buf = np.zeros(max(nbytes, 1), dtype=np.uint8)
        w = np.array([wf], dtype=np.int32)
        off = np.zeros(1, dtype=np.int64)
        self.check("gather", self.gather(pool.h, 1, w.ctypes.data, buf.ctypes.data, off.ctypes.data))
        return torch.from_numpy(buf[:nbytes].copy())

    def kv_staging(self, staging, device=None):
        staging = staging.cpu().numpy()
        return staging if staging.size else np.zeros(16, dtype=np.uint8)


def route_step_host(api, pool, wf, tok_off, tok, P, O, overhead, prefill, decode, qpen, alternates,
                    depth, limit, group=None):
    """paper_2603_13605_b200.dist.route_step over oracle pools: the oracle's match column, the
    product's exchange (dist.gather_columns, under gloo) and the oracle's cost batch."""
    import torch

    from paper_2603_13605_b200 import dist as sfdist
    wf = np.ascontiguousarray(wf, dtype=np.int32)
    tok_off = np.ascontiguousarray(tok_off, dtype=np.int64)
    par = [np.ascontiguousarray(x, dtype=np.float64) for x in (overhead, prefill, decode, qpen)]
    alt = None if alternates is None else np.ascontiguousarray(alternates, dtype=np.int32)
    P = np.ascontiguousarray(P, dtype=np.int64)
    O = np.ascontiguousarray(O, dtype=np.int64)
    depth = np.ascontiguousarray(depth, dtype=np.uint64).copy()
    R = len(wf)
    m_col = torch.from_numpy(pool.match(wf, tok_off, np.ascontiguousarray(tok, dtype=np.uint32)).astype(np.int64))
    M = np.ascontiguousarray(sfdist.gather_columns(m_col, group).numpy())
    world = M.shape[1]
    choice = np.zeros(R, np.int32)
    cost = np.zeros(R, np.float64)
    api.check("cost_batch", api.cost_batch(R, world, P.ctypes.data, M.ctypes.data, O.ctypes.data,
                                           *[x.ctypes.data for x in par], alt.ctypes.data if alt is not None else None,
                                           depth.ctypes.data, int(limit), choice.ctypes.data, cost.ctypes.data))
    return choice, cost, depth


def load():
    if "oracle" not in _cache:
        src = os.path.join(REPO, "oracle", "sfkv_oracle.c")
        if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=True)
        _cache["oracle"] = OracleApi(C.CDLL(ORACLE_SO))
    return _cache["oracle"]


def load_ref():
    """The reference's own functions, or None when oracle/_ref was not built here."""
    if "ref" not in _cache:
        _cache["ref"] = C.CDLL(REF_SO) if os.path.exists(REF_SO) else None
    return _cache["ref"]
