"""The drop-in, end to end: the reference's own Orchestrator + MemoryManager + harness loop drive
the B200 pool through GpuPinnedBackend (integration/, the reference-side binding of libsfkv), and
the result must equal the golden stream recorded from the unmodified reference on the same
(trace, config): every dispatch's (P, M) in event order, the full memory-manager action log
(trigger, ts, action, workflow, backend, reason) and the final backend counters.

Scenario inputs are written here: the reference demo parameters are restated as Python data (the
reference tree is absent on the GPU box) and the synthetic scenarios come from
tests/golden/make_golden.py's generators.
"""
import json
import os
import subprocess
import sys

import pytest

import replay

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(REPO, "oracle", "_ref", "sf_gpu_replay")
sys.path.insert(0, os.path.join(REPO, "tests", "golden"))

pytestmark = pytest.mark.gpu


def _sim(ref, model, tier, prefill, decode, maxc, cap, output, overhead=0.0):
    return {"ref": ref, "kind": "simulated", "model": model, "tier": tier,
            "sim": {"prefill_ms_per_token": prefill, "decode_ms_per_token": decode,
                    "fixed_overhead_ms": overhead, "max_concurrency": maxc,
                    "cache_capacity_tokens": cap, "output": output}}


MEM = {"chain": ["preserve_small_increment", "flush_at_boundary"], "tau": 512,
       "tau_pressure": 0.85, "monitor_interval_ms": 100}


def support_demo():
    script = {"rule": "script", "name": "customer_support"}
    cfg = {"label": "support-demo",
           "backends": [_sim("light", "sim-light-4b", "light", 1.0, 10.0, 2, 200000, script),
                        _sim("heavy", "sim-heavy-8b", "heavy", 2.0, 20.0, 2, 200000, script)],
           "mapper": {"type": "explicit"},
           "scheduling": {"stage_policy": "fcfs", "request_policy": "fcfs"},
           "memory": MEM,
           "templates": {"customer_support": {"light": "light", "heavy": "heavy",
                                              "tool_latency_ms": 40.0}}}
    tickets = [("My bill shows a duplicate charge for last month", "billing", "false"),
               ("The device will not power on after the update", "technical", "false"),
               ("I want to change my shipping address", "general", "false"),
               ("My account was accessed from another country", "technical", "true")]
    trace = [{"template": "customer_support", "arrival_ms": 50 * i,
              "payload": {"ticket": t, "category": c, "needs_escalation": e}}
             for i, (t, c, e) in enumerate(tickets)]
    return cfg, trace


def math_chain(override):
    cfg = {"label": "chain-" + override,
           "backends": [_sim("heavy", "sim-heavy-8b", "heavy", 2.0, 1.0, 1, 1000000,
                             {"rule": "constant", "tokens": 0})],
           "mapper": {"type": "explicit"}, "memory": MEM,
           "templates": {"math_chain_k": {"backend": "heavy", "k": 5, "base_tokens": 1000,
                                          "append_tokens": 50, "max_tokens": 256,
                                          "cache_override": override}}}
    trace = [{"template": "math_chain_k", "arrival_ms": a, "payload": {"base_tokens": 1000}}
             for a in (0, 10000)]
    return cfg, trace


def synthetic(name):
    import make_golden
    return getattr(make_golden, name)()


SCENARIOS = {
    "support_demo": support_demo,
    "chain_preserve": lambda: math_chain("none"),
    "chain_flush": lambda: math_chain("flush"),
    "alt_pressure": lambda: synthetic("alt_pressure"),
    "chain_scale": lambda: synthetic("chain_scale"),
}


@pytest.mark.parametrize("gpu_memory", [False, True], ids=["ref-memory", "gpu-memory"])
@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_reference_harness_on_gpu_pool_matches_golden(tmp_path, name, gpu_memory):
    """gpu-memory: the reference's MemoryManager is replaced by GpuMemoryManager (integration/),
    so pin cache, policy resolution, tracker and pressure ticks all run on the B200."""
    if not os.path.exists(DRIVER):
        pytest.fail("oracle/_ref/sf_gpu_replay missing: build it where /root/reference exists")
    cfg, trace = SCENARIOS[name]()
    cp, tp, op = tmp_path / "c.json", tmp_path / "t.jsonl", tmp_path / "o.jsonl"
    cp.write_text(json.dumps(cfg))
    tp.write_text("".join(json.dumps(r) + "\n" for r in trace))
    subprocess.run([DRIVER, "--config", str(cp), "--trace", str(tp), "--out", str(op)] +
                   (["--gpu-memory"] if gpu_memory else []), check=True, timeout=600)
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
