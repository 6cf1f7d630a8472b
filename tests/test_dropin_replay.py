"""The drop-in, end to end: the reference's own Orchestrator + MemoryManager + harness loop drive
the B200 pool through GpuPinnedBackend (integration/, the reference-side binding of libsfkv), and
the result must equal the golden stream recorded from the unmodified reference on the same
(trace, config): every dispatch's (P, M) in event order, the full memory-manager action log
(trigger, ts, action, workflow, backend, reason) and the final backend counters.

Scenario inputs come from tests/dropin_scenarios.py (shared with bench.py's C1 leg).
"""
import json
import os
import subprocess

import pytest

import replay
from dropin_scenarios import FLAGS, SCENARIOS

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(REPO, "oracle", "_ref", "sf_gpu_replay")

pytestmark = pytest.mark.gpu


MODES = {"ref-memory": [], "gpu-memory": ["--gpu-memory"], "gpu-all": ["--gpu-memory", "--gpu-router"],
         "host-tokenizer": ["--host-tokenizer"]}


@pytest.mark.parametrize("mode", sorted(MODES))
@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_reference_harness_on_gpu_pool_matches_golden(tmp_path, name, mode):
    """Every mode tokenizes and interns on the GPU (sfkv_tokenize_batch, one batch per dispatch
    instant) except host-tokenizer (context_token_sequence + a host string map).
    gpu-memory: the reference's MemoryManager is replaced by GpuMemoryManager (integration/),
    so pin cache, policy resolution, tracker and pressure ticks all run on the B200; gpu-all also
    replaces the stage routers (integration/gpu_router.hpp: plan / threshold / one-bit decisions
    and reroute_on_overload through sfmap_*)."""
    if not os.path.exists(DRIVER):
        pytest.fail("oracle/_ref/sf_gpu_replay missing: build it where /root/reference exists")
    cfg, trace = SCENARIOS[name]()
    cp, tp, op = tmp_path / "c.json", tmp_path / "t.jsonl", tmp_path / "o.jsonl"
    cp.write_text(json.dumps(cfg))
    tp.write_text("".join(json.dumps(r) + "\n" for r in trace))
    subprocess.run([DRIVER, "--config", str(cp), "--trace", str(tp), "--out", str(op)] +
                   MODES[mode] + FLAGS.get(name, []), check=True, timeout=600)
    got = [json.loads(l) for l in op.read_text().splitlines()]
    gold = replay.load_stream(name)

    want_req = [(l["b"], l["wf"], l["stage"], l["P"], l["M"]) for l in gold if l.get("op") == "match"]
    got_req = [(l["b"], l["wf"], l["stage"], l["P"], l["M"]) for l in got if l["type"] == "req"]
    assert got_req == want_req

    keys = ("trigger", "ts", "action", "workflow", "backend", "reason")
    want_act = [tuple(l[k] for k in keys) for l in gold if l["type"] == "act"]
    got_act = [tuple(l[k] for k in keys) for l in got if l["type"] == "act"]
    assert got_act == want_act

    gend = next(l for l in gold if l["type"] == "end")
    oend = next(l for l in got if l["type"] == "end")
    assert oend["now_ms"] == gend["now_ms"]
    for ref, want in gend["backends"].items():
        assert oend["backends"][ref] == want, ref
