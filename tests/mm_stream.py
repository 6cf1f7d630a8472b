"""Memory-manager signal streams for the tracker parity tests (test infrastructure).

* `GoldenWalk` replays a golden stream's lifecycle signals and pressure ticks (recorded from the
  reference by oracle/_ref/sf_ref_replay, tests/golden/) through a `Tracker` — batched between
  ticks — and rebuilds the MemoryManager action log (trigger, ts, action, workflow, backend,
  reason) to compare with the reference's own records.
* `random_stream` generates seeded signal streams with concurrency, overrides, per-workflow
  chains, pressure ticks and deliberately out-of-order signals.
* `RefManager` drives the reference's MemoryManager (oracle/_ref/libsfref.so) with the same
  stream, one on_signal call at a time.
Interning follows the drop-in's rules: backends in sorted-ref order (BackendRegistry::refs),
workflow slots in first-seen order with ranks from workflow-id string order, dense stage ids per
workflow, dense model ids.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2603_13605_b200.abi import MM_ACT, MM_OVERRIDE, MM_REASON

KIND = {"stage_start": 0, "stage_complete": 1, "workflow_complete": 2}
KIND_NAME = {v: k for k, v in KIND.items()}


class Interner:
    def __init__(self, backends, workflows):
        self.backends = sorted(backends)
        self.bidx = {b: i for i, b in enumerate(self.backends)}
        self.wf = {}
        self.stages = {}
        self.models = {}
        order = sorted(set(workflows))
        self.rank_of = {w: i for i, w in enumerate(order)}

    def w(self, wf):
        if wf not in self.wf:
            self.wf[wf] = len(self.wf)
            self.stages[wf] = {}
        return self.wf[wf]

    def s(self, wf, st):
        d = self.stages[wf]
        if st not in d:
            d[st] = len(d)
        return d[st]

    def m(self, model):
        return self.models.setdefault(model, len(self.models))

    def ranks(self, n):
        r = np.zeros(n, np.uint32)
        for wf, slot in self.wf.items():
            r[slot] = self.rank_of[wf]
        return r


def encode(intern, sigs):
    """List of signal dicts -> SoA arrays for Tracker.on_signals."""
    n = len(sigs)
    kind = np.zeros(n, np.uint8)
    wf = np.zeros(n, np.int32)
    stage = np.zeros(n, np.int32)
    backend = np.zeros(n, np.int32)
    model = np.zeros(n, np.int32)
    tokens = np.zeros(n, np.int64)
    ts = np.zeros(n, np.float64)
    ov = np.zeros(n, np.uint8)
    for i, s in enumerate(sigs):
        kind[i] = KIND[s["kind"]]
        wf[i] = intern.w(s["wf"])
        ts[i] = s["ts"]
        if s["kind"] != "workflow_complete":
            stage[i] = intern.s(s["wf"], s["stage"])
            backend[i] = intern.bidx[s["b"]]
            model[i] = intern.m(s["model"])
            tokens[i] = s["tokens"]
            ov[i] = MM_OVERRIDE[s.get("override", "none")]
    return kind, wf, stage, backend, model, tokens, ts, ov


def trigger_of(s):
    t = f"{s['kind']} {s['wf']}"
    return t + (f"/{s['stage']}" if s.get("stage") else "")


def records_to_log(intern, sigs, out):
    """Tracker outputs of a batch -> (log records, statuses)."""
    cnt, st, k, b, r = out
    log = []
    for i, s in enumerate(sigs):
        for j in range(int(cnt[i])):
            act = MM_ACT[int(k[i, j])]
            noop = act == "noop"
            log.append({"trigger": trigger_of(s), "ts": float(s["ts"]), "action": act,
                        "workflow": "" if noop else s["wf"],
                        "backend": "" if noop else intern.backends[int(b[i, j])],
                        "reason": MM_REASON[int(r[i, j])]})
    return log, [int(x) for x in st]


def tick_log(intern, victims, ts):
    inv = {v: k for k, v in intern.wf.items()}
    log = []
    for bi, w in enumerate(victims):
        if w >= 0:
            log.append({"trigger": "pressure_tick", "ts": float(ts), "action": "flush",
                        "workflow": inv[int(w)], "backend": intern.backends[bi],
                        "reason": "flush_under_pressure"})
    return log


def failed_flushes(out, flaky, backends):
    """(wf slot, backend, signal index) of every flush record a backend refused twice: apply_action
    retries once (memory.cpp:189-203), so only mode 2 (every attempt fails) gives up; mode 1 (the
    first attempt of each flush fails) succeeds on the retry."""
    cnt, st, k, b, r = out
    res = []
    for i in range(len(cnt)):
        for j in range(int(cnt[i])):
            if int(k[i, j]) == 1 and flaky.get(backends[int(b[i, j])], 0) == 2:
                res.append((i, int(b[i, j])))
    return res


def run_stream(tracker, intern, events, batch_between_ticks=True, flaky=None):
    """events: ("sig", dict) / ("tick", {"util": {ref: u}, "ts": t}). Returns (log, statuses).
    flaky: {backend ref: mode} of backends whose flush throws (see failed_flushes); the host
    reports the flushes that failed twice back to the tracker (sfmm_flush_failed)."""
    log, statuses, batch = [], [], []
    flaky = flaky or {}

    def flush_batch():
        if not batch:
            return
        tracker.set_ranks(intern.ranks(tracker.W))
        enc = encode(intern, batch)
        out = tracker.on_signals(*enc)
        bad = failed_flushes(out, flaky, intern.backends)
        if bad:
            tracker.flush_failed([enc[1][i] for i, _ in bad], [bb for _, bb in bad], [i for i, _ in bad])
        l, st = records_to_log(intern, batch, out)
        log.extend(l)
        statuses.extend(st)
        batch.clear()

    for kind, ev in events:
        if kind == "sig":
            for wf in [ev["wf"]]:
                intern.w(wf)
            if ev.get("chain") is not None:  # set_workflow_chain before the first signal
                flush_batch()
                tracker.set_chain(intern.w(ev["wf"]), ev["chain"])
            batch.append(ev)
            if not batch_between_ticks:
                flush_batch()
        else:
            flush_batch()
            tracker.set_ranks(intern.ranks(tracker.W))
            util = np.array([ev["util"].get(b, 0.0) for b in intern.backends], np.float64)
            victims = tracker.pressure_tick(util)
            bad = [(int(w), bi) for bi, w in enumerate(victims)
                   if w >= 0 and flaky.get(intern.backends[bi], 0) == 2]
            if bad:
                tracker.flush_failed([w for w, _ in bad], [bi for _, bi in bad], [-1] * len(bad))
            log.extend(tick_log(intern, victims, ev["ts"]))
    flush_batch()
    return log, statuses


# ---------------------------------------------------------------- golden streams -----------
def golden_events(lines):
    meta = next(l for l in lines if l.get("type") == "meta")
    recs = sorted((l for l in lines if l.get("type") in ("sig", "tick")), key=lambda l: l["seq"])
    events = [("sig", l) if l["type"] == "sig" else ("tick", l) for l in recs]
    acts = [l for l in lines if l.get("type") == "act"]
    backends = [b["ref"] for b in meta["backends"]]
    wfs = [l["wf"] for l in lines if l.get("type") == "sig"]
    return meta, events, acts, backends, wfs


# ---------------------------------------------------------------- random streams -----------
def random_stream(seed, n_wf=40, backends=("A", "B", "C"), models=("m1", "m2"), n_stages=(1, 6),
                  p_override=0.1, p_chain=0.2, p_bad=0.03, p_tick=0.05, tau=512, chain_len=(1, 4)):
    """Seeded lifecycle-signal stream with concurrency and deliberate order violations."""
    rng = np.random.default_rng(seed)
    plans = {}
    for w in range(n_wf):
        wid = f"wf-{rng.integers(0, 10**6):06d}-{w}"
        k = int(rng.integers(n_stages[0], n_stages[1] + 1))
        toks = int(rng.integers(0, 3000))
        stages = []
        for s in range(k):
            toks += int(rng.choice([0, rng.integers(1, tau), rng.integers(tau, 3 * tau)]))
            stages.append({"stage": f"s{s}", "b": str(rng.choice(backends)), "model": str(rng.choice(models)),
                           "tokens": toks, "override": str(rng.choice(["none", "flush", "preserve"],
                                                                     p=[1 - p_override, p_override / 2, p_override / 2]))})
        chain = None
        if rng.random() < p_chain:
            chain = [str(x) for x in rng.choice(["preserve_small_increment", "flush_at_boundary"],
                                                size=int(rng.integers(*chain_len)))]
        plans[wid] = {"stages": stages, "next": 0, "open": [], "done": False, "chain": chain,
                      "first": True}
    events, ts = [], 0.0
    active = list(plans)
    while active:
        ts += float(rng.choice([0.0, 0.5, 1.0, 7.0]))
        if rng.random() < p_tick:
            events.append(("tick", {"util": {b: float(rng.choice([0.2, 0.86, 0.9, 1.0])) for b in backends},
                                    "ts": ts}))
            continue
        wid = str(rng.choice(active))
        p = plans[wid]
        sig = None
        if rng.random() < p_bad:  # an out-of-order signal
            s = p["stages"][int(rng.integers(0, len(p["stages"])))]
            kind = str(rng.choice(["stage_start", "stage_complete", "workflow_complete"]))
            sig = {"kind": kind, "wf": wid, "stage": "" if kind == "workflow_complete" else s["stage"],
                   "b": str(rng.choice(backends)), "model": s["model"], "tokens": s["tokens"],
                   "override": "none"}
        else:
            can_start = p["next"] < len(p["stages"]) and (not p["open"] or rng.random() < 0.4)
            if can_start and (not p["open"] or rng.random() < 0.5):
                s = p["stages"][p["next"]]
                p["next"] += 1
                p["open"].append(s)
                sig = dict(kind="stage_start", wf=wid, **s)
            elif p["open"]:
                s = p["open"].pop(int(rng.integers(0, len(p["open"]))))
                done = dict(s)
                done["tokens"] = s["tokens"] + int(rng.integers(0, 50)) if rng.random() < 0.8 else 0
                sig = dict(kind="stage_complete", wf=wid, **{k: v for k, v in done.items()})
            else:
                sig = {"kind": "workflow_complete", "wf": wid, "stage": "", "b": "", "model": "",
                       "tokens": 0, "override": "none"}
                active.remove(wid)
        sig["ts"] = ts
        if p["first"]:
            sig["chain"] = p["chain"]
            p["first"] = False
        events.append(("sig", sig))
    return events, list(backends), list(plans)


class RefManager:
    """The reference's MemoryManager through oracle/_ref/libsfref.so."""

    def __init__(self, tau, tau_pressure, chain, flaky=None, backends=()):
        """flaky: {ref: mode} -> a BackendRegistry of test backends over `backends` whose flush
        throws (sfref_mm_create_flaky); None -> no registry (every action applies)."""
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                            "libsfref.so")
        L = C.CDLL(path)
        L.sfref_mm_create.restype = C.c_void_p
        L.sfref_mm_create.argtypes = [C.c_longlong, C.c_double, C.c_int, C.POINTER(C.c_char_p)]
        L.sfref_mm_create_flaky.restype = C.c_void_p
        L.sfref_mm_create_flaky.argtypes = [C.c_longlong, C.c_double, C.c_int, C.POINTER(C.c_char_p), C.c_int,
                                            C.POINTER(C.c_char_p), C.POINTER(C.c_int)]
        L.sfref_mm_entry.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p]
        L.sfref_mm_destroy.argtypes = [C.c_void_p]
        L.sfref_mm_set_chain.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_char_p)]
        L.sfref_mm_on_signal.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_char_p, C.c_char_p,
                                         C.c_char_p, C.c_longlong, C.c_double, C.c_int]
        L.sfref_mm_pressure_tick.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_char_p),
                                             C.POINTER(C.c_double), C.c_double]
        L.sfref_mm_log_size.restype = C.c_longlong
        L.sfref_mm_log_size.argtypes = [C.c_void_p]
        L.sfref_mm_log_get.argtypes = [C.c_void_p, C.c_longlong, C.POINTER(C.c_int), C.c_char_p,
                                       C.c_char_p, C.c_char_p, C.c_char_p, C.c_int,
                                       C.POINTER(C.c_double)]
        self.L = L
        arr = (C.c_char_p * len(chain))(*[c.encode() for c in chain])
        if flaky is None:
            self.h = L.sfref_mm_create(tau, tau_pressure, len(chain), arr)
        else:
            refs = sorted(backends)
            ra = (C.c_char_p * len(refs))(*[r.encode() for r in refs])
            ma = (C.c_int * len(refs))(*[int(flaky.get(r, 0)) for r in refs])
            self.h = L.sfref_mm_create_flaky(tau, tau_pressure, len(chain), arr, len(refs), ra, ma)

    def entry(self, wf, backend):
        """0 absent, 1 present + preserved, 2 present unpreserved (WorkflowTracker::entry)."""
        return self.L.sfref_mm_entry(self.h, wf.encode(), backend.encode())

    def close(self):
        if self.h:
            self.L.sfref_mm_destroy(self.h)
            self.h = None

    def run(self, events, backends):
        statuses = []
        refs = sorted(backends)
        for kind, ev in events:
            if kind == "sig":
                if ev.get("chain"):
                    arr = (C.c_char_p * len(ev["chain"]))(*[c.encode() for c in ev["chain"]])
                    self.L.sfref_mm_set_chain(self.h, ev["wf"].encode(), len(ev["chain"]), arr)
                st = self.L.sfref_mm_on_signal(
                    self.h, KIND[ev["kind"]], ev["wf"].encode(), ev.get("stage", "").encode(),
                    ev.get("b", "").encode(), ev.get("model", "").encode(), int(ev.get("tokens", 0)),
                    float(ev["ts"]), MM_OVERRIDE[ev.get("override", "none")])
                statuses.append(st)
            else:
                r = (C.c_char_p * len(refs))(*[b.encode() for b in refs])
                u = (C.c_double * len(refs))(*[ev["util"].get(b, 0.0) for b in refs])
                self.L.sfref_mm_pressure_tick(self.h, len(refs), r, u, float(ev["ts"]))
        log = []
        buf = [C.create_string_buffer(512) for _ in range(4)]
        k, ts = C.c_int(), C.c_double()
        for i in range(self.L.sfref_mm_log_size(self.h)):
            self.L.sfref_mm_log_get(self.h, i, C.byref(k), *buf, 512, C.byref(ts))
            log.append({"trigger": buf[3].value.decode(), "ts": ts.value, "action": MM_ACT[k.value],
                        "workflow": buf[0].value.decode(), "backend": buf[1].value.decode(),
                        "reason": buf[2].value.decode()})
        return log, statuses
