"""Batched MemoryManager (§8f-1): the tracker restatement against the reference.

CPU: the oracle tracker (oracle/sfkv_oracle.c, sfo_tracker_*) reproduces (1) every golden
stream's action log — trigger, ts, action, workflow, backend, reason, in order, pressure ticks
included — recorded from the reference harness, and (2) the reference's own MemoryManager
(oracle/_ref/libsfref.so) on seeded random streams with overrides, per-workflow chains,
concurrent stages, pressure ticks and out-of-order signals, one signal at a time.
GPU (`-m gpu`): the sm_100a tracker (sfmm_*) equals the oracle on the same streams in large
batches (parallel across workflows) and reproduces the golden logs."""
import os

import pytest

import replay
from mm_stream import Interner, RefManager, golden_events, random_stream, run_stream
from paper_2603_13605_b200.abi import Tracker

REF_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "libsfref.so")


def _golden(api, name, batched, device=0):
    lines = replay.load_stream(name)
    meta, events, acts, backends, wfs = golden_events(lines)
    intern = Interner(backends, wfs)
    tr = Tracker(api, max_workflows=len(set(wfs)) + 1, n_backends=len(backends), chain=meta["chain"],
                 tau=meta["tau"], tau_pressure=meta["tau_pressure"], device=device)
    log, statuses = run_stream(tr, intern, events, batch_between_ticks=batched, flaky=meta.get("flaky"))
    tr.close()
    want = [{k: a[k] for k in ("trigger", "ts", "action", "workflow", "backend", "reason")} for a in acts]
    return log, want, statuses


@pytest.mark.parametrize("name", replay.stream_names())
@pytest.mark.parametrize("batched", [False, True])
def test_oracle_tracker_reproduces_golden_action_log(oracle_api, name, batched):
    log, want, statuses = _golden(oracle_api, name, batched)
    assert all(s == 0 for s in statuses)
    assert log == want


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_oracle_tracker_matches_reference_memory_manager(oracle_api, seed):
    events, backends, wfs = random_stream(seed)
    chain = ["preserve_small_increment", "flush_at_boundary"] if seed % 2 else ["flush_at_boundary"]
    ref = RefManager(512, 0.85, chain)
    want_log, want_st = ref.run(events, backends)
    ref.close()
    intern = Interner(backends, wfs)
    tr = Tracker(oracle_api, max_workflows=len(wfs), n_backends=len(backends), chain=chain)
    log, st = run_stream(tr, intern, events, batch_between_ticks=False)
    assert st == want_st
    assert any(s != 0 for s in st), "stream should exercise out-of-order signals"
    assert log == want_log


def _entry_states(tr, intern, backends, wfs):
    """WorkflowTracker::entry per (workflow, backend): 0 absent, 1 preserved, 2 unpreserved."""
    pres, keep = tr.entries()[:2]
    out = {}
    for w in sorted(set(wfs)):
        for b in backends:
            if w not in intern.wf:
                out[(w, b)] = 0
                continue
            s, bi = intern.wf[w], intern.bidx[b]
            out[(w, b)] = 0 if not pres[s, bi] else (1 if keep[s, bi] else 2)
    return out


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [21, 22, 23, 24])
@pytest.mark.parametrize("cut", [0.4, 0.7, 1.0])
def test_oracle_tracker_failure_path_matches_reference(oracle_api, seed, cut):
    """apply_action's failure branch (memory.cpp:189-203, 319-325): backend B's flush always
    throws (entries stay, unpreserved), C's fails once then succeeds on the retry. The reference
    MemoryManager runs over a registry of those test backends; the oracle tracker gets the failed
    flushes reported back (sfo_flush_failed). Logs, statuses and every tracker entry agree."""
    backends = ("A", "B", "C")
    flaky = {"B": 2, "C": 1}
    events, _, wfs = random_stream(seed, n_wf=60, backends=backends, p_tick=0.08, p_override=0.25)
    events = events[: int(len(events) * cut)]  # tracker state mid-stream (workflows still live)
    chain = ["preserve_small_increment", "flush_at_boundary"]
    ref = RefManager(512, 0.85, chain, flaky=flaky, backends=backends)
    want_log, want_st = ref.run(events, backends)
    want_entries = {(w, b): ref.entry(w, b) for w in sorted(set(wfs)) for b in backends}
    ref.close()
    intern = Interner(backends, wfs)
    tr = Tracker(oracle_api, max_workflows=len(set(wfs)), n_backends=len(backends), chain=chain)
    log, st = run_stream(tr, intern, events, batch_between_ticks=False, flaky=flaky)
    assert st == want_st
    assert log == want_log
    got = _entry_states(tr, intern, backends, wfs)
    assert got == want_entries
    if cut < 1:
        assert 2 in want_entries.values(), "the stream should leave unpreserved entries behind"


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [31, 32])
def test_oracle_tracker_many_stages_and_long_chains_match_reference(oracle_api, seed):
    """No caps: workflows with 70-140 stages (stage ids past 64 and past 128) and per-workflow
    policy chains of 9-15 entries, against the reference MemoryManager."""
    events, backends, wfs = random_stream(seed, n_wf=12, n_stages=(70, 140), p_chain=0.6, chain_len=(9, 16),
                                          p_tick=0.02)
    chain = ["flush_at_boundary"] * 3 + ["preserve_small_increment"] * 7  # a 10-entry default chain
    ref = RefManager(512, 0.85, chain)
    want_log, want_st = ref.run(events, backends)
    ref.close()
    intern = Interner(backends, wfs)
    tr = Tracker(oracle_api, max_workflows=len(wfs), n_backends=len(backends), chain=chain, max_stages=32)
    tr.reserve(max_stages=160)
    log, st = run_stream(tr, intern, events, batch_between_ticks=False)
    assert st == want_st
    assert log == want_log


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [21, 22])
def test_gpu_tracker_failure_path_matches_oracle(gpu_api, oracle_api, seed):
    """The same failure-path streams on the GPU in large batches (failed flushes reported per
    batch with their signal index)."""
    backends = ("A", "B", "C")
    flaky = {"B": 2, "C": 1}
    events, _, wfs = random_stream(seed, n_wf=400, backends=backends, p_tick=0.01, p_override=0.25)
    events = events[: len(events) * 2 // 3]
    out = []
    for api in (oracle_api, gpu_api):
        intern = Interner(backends, wfs)
        tr = Tracker(api, max_workflows=len(set(wfs)), n_backends=len(backends))
        log, st = run_stream(tr, intern, events, batch_between_ticks=True, flaky=flaky)
        out.append((log, st, _entry_states(tr, intern, backends, wfs)))
        tr.close()
    assert out[0] == out[1]


@pytest.mark.gpu
def test_gpu_tracker_grows_and_long_chains_match_oracle(gpu_api, oracle_api):
    """Stage ids past 64 (global stage words), 10-entry chains and growth mid-stream: the GPU
    tracker starts with 8 slots / 64 stages and is reserved up between batches."""
    events, backends, wfs = random_stream(33, n_wf=300, n_stages=(60, 100), p_chain=0.5, chain_len=(9, 12),
                                          p_tick=0.002)
    chain = ["flush_at_boundary"] * 4 + ["preserve_small_increment"] * 6
    out = []
    for api in (oracle_api, gpu_api):
        intern = Interner(backends, wfs)
        tr = Tracker(api, max_workflows=8, n_backends=len(backends), chain=chain)
        tr.reserve(max_workflows=len(set(wfs)), max_stages=128)
        log, st = run_stream(tr, intern, events, batch_between_ticks=True)
        out.append((log, st, [e.copy() for e in tr.entries()]))
        tr.close()
    (lo, so, eo), (lg, sg, eg) = out
    assert sg == so and lg == lo
    for a, b in zip(eo, eg):
        assert (a == b).all()


@pytest.mark.gpu
@pytest.mark.parametrize("name", replay.stream_names())
def test_gpu_tracker_reproduces_golden_action_log(gpu_api, name):
    log, want, statuses = _golden(gpu_api, name, batched=True)
    assert all(s == 0 for s in statuses)
    assert log == want


@pytest.mark.gpu
@pytest.mark.parametrize("seed,n_wf,nb", [(11, 60, 5), (12, 500, 5), (13, 3000, 5), (14, 400, 12)])
def test_gpu_tracker_matches_oracle_in_large_batches(gpu_api, oracle_api, seed, n_wf, nb):
    """nb = 12 backends exercises the replay with (wf, b) entries in global memory (the
    thread-local cache covers <= 8)."""
    events, backends, wfs = random_stream(seed, n_wf=n_wf, backends=tuple("ABCDEFGHIJKL"[:nb]),
                                          p_tick=0.002)
    out = []
    for api in (oracle_api, gpu_api):
        intern = Interner(backends, wfs)
        tr = Tracker(api, max_workflows=len(wfs), n_backends=len(backends))
        log, st = run_stream(tr, intern, events, batch_between_ticks=True)
        out.append((log, st, tr.entries()))
        tr.close()
    (lo, so, eo), (lg, sg, eg) = out
    assert sg == so
    assert lg == lo
    for a, b in zip(eo, eg):  # tracker state after the stream
        assert (a == b).all()


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [7, 8])
def test_action_log_jsonl_byte_identical_to_reference_export(oracle_api, seed):
    """§8f-4: the JSONL the GPU path writes (paper_2603_13605_b200.sim_server.action_log_jsonl over
    the tracker's records) equals MemoryManager::export_action_log byte for byte."""
    import ctypes as C

    from paper_2603_13605_b200.sim_server import action_log_jsonl
    events, backends, wfs = random_stream(seed)
    chain = ["preserve_small_increment", "flush_at_boundary"]
    ref = RefManager(512, 0.85, chain)
    ref.run(events, backends)
    L = ref.L
    L.sfref_mm_export.restype = C.c_longlong
    L.sfref_mm_export.argtypes = [C.c_void_p, C.c_char_p, C.c_longlong]
    n = L.sfref_mm_export(ref.h, None, 0)
    buf = C.create_string_buffer(n + 1)
    L.sfref_mm_export(ref.h, buf, n + 1)
    want = buf.raw[:n].decode()
    ref.close()
    tr = Tracker(oracle_api, max_workflows=len(wfs), n_backends=len(backends), chain=chain)
    log, _ = run_stream(tr, Interner(backends, wfs), events, batch_between_ticks=False)
    got = action_log_jsonl(log)
    assert got.count("\n") > 100
    assert got == want
