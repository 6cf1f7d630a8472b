"""Drop-in scenarios (SURVEY §8d C1 and the synthetic ones): reference-format configs and traces
for the reference's harness, shared by tests/test_dropin_replay.py and bench.py's C1 leg. The
reference demo parameters (proj/configs/support_demo.json, proj/traces/support_demo.jsonl;
mapped_one_bit.json x mixed_workload.jsonl in make_golden.py) are restated as Python data because
the reference tree is absent on the GPU box; the synthetic scenarios come from
tests/golden/make_golden.py's generators."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))


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
    "alt_pressure_flaky": lambda: synthetic("alt_pressure"),
    "chain_scale_flaky": lambda: synthetic("chain_scale"),
    "mapped_one_bit": lambda: synthetic("mapped_one_bit"),
    "mapped_one_bit_reroute": lambda: synthetic("mapped_one_bit_reroute"),
    "mapped_threshold_reroute": lambda: synthetic("mapped_threshold_reroute"),
}
# Driver flags of the failure-path scenarios (make_golden.FLAKY: backends whose flush throws).
FLAGS = {"alt_pressure_flaky": ["--flaky", "A:1,B:2"], "chain_scale_flaky": ["--flaky", "heavy:2"]}
