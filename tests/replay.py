"""Replays a golden stream (tests/golden/*.jsonl.gz, recorded from the unmodified reference) through
an sfkv-ABI implementation — the GPU library or the CPU oracle — and checks every Class A output:
per-request M, pin admission, occupancy after every pin/flush, flush freed tokens, preserve
results, utilization values (exact doubles), pressure-tick victims, and the final counters.

Batched mode groups runs of consecutive match ops (and of pin ops on distinct workflows) per
backend into one batch call, which is how the GPU path is meant to be driven; the sequence of
observable results must not change.
"""
from __future__ import annotations

import gzip
import json
import os

import numpy as np

from paper_2603_13605_b200.abi import BLOCK_TOKENS, Config, Pool, csr

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_stream(name):
    with gzip.open(os.path.join(GOLDEN, f"{name}.jsonl.gz"), "rt") as f:
        return [json.loads(line) for line in f]


def stream_names():
    return sorted(f[: -len(".jsonl.gz")] for f in os.listdir(GOLDEN) if f.endswith(".jsonl.gz"))


class Mismatch(AssertionError):
    pass


def _eq(what, got, want, rec):
    if got != want:
        raise Mismatch(f"{what}: got {got!r}, reference {want!r} at seq {rec.get('seq')}: "
                       f"{ {k: v for k, v in rec.items() if k != 'tok'} }")


def pool_config_for(lines, ref, n_slabs=0, slab_row_bytes=0, device=0):
    meta = lines[0]
    be = next(b for b in meta["backends"] if b["ref"] == ref)
    wfs = {l["wf"] for l in lines if l.get("b") == ref and "wf" in l}
    max_p = max([l["P"] for l in lines if l.get("op") == "match" and l.get("b") == ref] + [1])
    mpb = (max_p + BLOCK_TOKENS - 1) // BLOCK_TOKENS + 1
    cap = int(be["capacity_tokens"])
    n_blocks = cap // BLOCK_TOKENS + len(wfs) + 2 * mpb + 64
    tl = 10
    while (1 << tl) < 2 * n_blocks:
        tl += 1
    return Config(max_workflows=len(wfs) + 1, n_blocks=n_blocks, capacity_tokens=cap,
                  max_pin_blocks=mpb, table_log2=tl, n_slabs=n_slabs,
                  slab_row_bytes=slab_row_bytes, device=device)


def replay(lines, api, pressure=None, batched=False, device=0, tokens=None):
    """pressure: callable(entries..) -> victims, defaults to api.pressure_argmin.
    tokens: the u32 token file of a stream recorded with --tok-out (match records carry "toff"
    instead of inline "tok")."""
    meta = lines[0]
    assert meta["type"] == "meta"
    refs = [b["ref"] for b in meta["backends"]]
    pools = {r: Pool(api, pool_config_for(lines, r, device=device)) for r in refs}
    slots = {r: {} for r in refs}
    toks = {r: {} for r in refs}

    def slot(ref, wf):
        m = slots[ref]
        if wf not in m:
            m[wf] = len(m)
        return m[wf]

    pending = {r: [] for r in refs}  # batched mode: queued match or pin records

    def drain(ref):
        q = pending[ref]
        if not q:
            return
        kind = q[0]["op"]
        pool = pools[ref]
        seqs = [toks[ref][l["rid"]] for l in q]
        off, tok = csr(seqs)
        wf = np.array([slot(ref, l["wf"]) for l in q], dtype=np.int32)
        if kind == "match":
            M = pool.match(wf, off, tok)
            for l, m in zip(q, M):
                _eq("M", int(m), l["M"], l)
        else:
            st = pool.commit(wf, off, tok)
            for l, s in zip(q, st):
                _eq("pin accepted", bool(s), l["accepted"], l)
            _eq("occupancy", pool.stats()["occupancy_tokens"], q[-1]["occ"], q[-1])
        pending[ref] = []

    n_checked = 0
    for l in lines[1:]:
        t = l["type"]
        if t == "op":
            ref, op = l["b"], l["op"]
            pool = pools[ref]
            if op == "match":
                if "tok" not in l:
                    l["tok"] = tokens[l["toff"]:l["toff"] + l["P"]]
                toks[ref][l["rid"]] = l["tok"]
            if batched and op in ("match", "pin"):
                q = pending[ref]
                if q and (q[0]["op"] != op or (op == "pin" and any(x["wf"] == l["wf"] for x in q))):
                    drain(ref)
                pending[ref].append(l)
                n_checked += 1
                continue
            drain(ref)
            if op == "match":
                off, tok = csr([l["tok"]])
                M = pool.match(np.array([slot(ref, l["wf"])], dtype=np.int32), off, tok)
                _eq("M", int(M[0]), l["M"], l)
            elif op == "pin":
                off, tok = csr([toks[ref][l["rid"]]])
                st = pool.commit(np.array([slot(ref, l["wf"])], dtype=np.int32), off, tok)
                _eq("pin accepted", bool(st[0]), l["accepted"], l)
                _eq("occupancy", pool.stats()["occupancy_tokens"], l["occ"], l)
            elif op == "flush":
                freed = pool.flush(-1 if l["all"] else slot(ref, l["wf"]))
                _eq("flush freed", freed, l["freed"], l)
                _eq("occupancy", pool.stats()["occupancy_tokens"], l["occ"], l)
            elif op == "preserve":
                _eq("preserve", pool.preserve(slot(ref, l["wf"])), l["ret"], l)
            elif op == "util":
                _eq("utilization", pool.cache_utilization(), l["value"], l)
            n_checked += 1
        elif t == "tick":
            for r in refs:
                drain(r)
            entries = l["entries"]
            if entries:
                names = sorted({e[0] for e in entries}, key=lambda s: s.encode())
                rank = {w: i for i, w in enumerate(names)}
                bidx = {r: i for i, r in enumerate(refs)}
                backend = np.array([bidx[e[1]] for e in entries], dtype=np.int32)
                ts = np.array([e[2] for e in entries], dtype=np.float64)
                wr = np.array([rank[e[0]] for e in entries], dtype=np.uint32)
                inf = np.array([e[3] for e in entries], dtype=np.int32)
                pres = np.ones(len(entries), dtype=np.uint8)
                util = np.array([l["util"][r] for r in refs], dtype=np.float64)
                victims = (pressure or default_pressure(api, device))(
                    backend, ts, wr, inf, pres, util, meta["tau_pressure"])
                got = sorted((entries[v][0], refs[b]) for b, v in enumerate(victims) if v >= 0)
            else:
                got = []
            want = sorted(tuple(v) for v in l["victims"])
            _eq("pressure victims", got, want, l)
            n_checked += 1
        elif t == "end":
            for r in refs:
                drain(r)
            for r, want in l["backends"].items():
                s = pools[r].stats()
                _eq(f"{r} occupancy", s["occupancy_tokens"], want["occupancy_tokens"], l)
                _eq(f"{r} capacity_rejections", s["capacity_rejections"],
                    want["capacity_rejections"], l)
                _eq(f"{r} flush_calls", s["flush_calls"], want["flush_calls"], l)
                _eq(f"{r} preserve_calls", s["preserve_calls"], want["preserve_calls"], l)
                _eq(f"{r} utilization", pools[r].cache_utilization(), want["utilization"], l)
    for p in pools.values():
        p.close()
    return n_checked


def default_pressure(api, device=0):
    def run(backend, ts, wr, inf, pres, util, tau):
        out = np.full(len(util), -1, dtype=np.int64)
        args = [len(backend), backend.ctypes.data, ts.ctypes.data, wr.ctypes.data,
                inf.ctypes.data, pres.ctypes.data, len(util), util.ctypes.data, tau,
                out.ctypes.data]
        api.check("pressure_argmin", api.dev_call("pressure_argmin", device, *args))
        return out
    return run
