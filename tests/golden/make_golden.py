"""Regenerate the golden streams under tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs /root/reference and oracle/_ref/sf_ref_replay):

    make -C oracle ref && python tests/golden/make_golden.py

Each stream is the reference's own replay of a (trace, config) pair, recorded by
oracle/ref_shim/replay_driver.cpp: every prefix_match / pin_prompt / flush / preserve /
cache_utilization call in event order, the lifecycle signals, the tracker snapshot and verdict of
every pressure tick, the memory manager's action log and the final backend counters.

Scenarios:
  support_demo      proj/traces/support_demo.jsonl x proj/configs/support_demo.json     (config C1)
  chain_preserve    proj/traces/math_chain.jsonl   x proj/configs/chain_preserve.json
  chain_flush       proj/traces/math_chain.jsonl   x proj/configs/chain_flush.json
  mapped_one_bit    proj/traces/mixed_workload.jsonl x proj/configs/mapped_one_bit.json
  single_heavy      proj/traces/mixed_workload.jsonl x proj/configs/single_heavy.json
  alt_pressure      synthetic, SURVEY §9 C4 probe 2 at 1/64 scale: A->B->A->B workflows under
                    chain [preserve_small_increment]; pressure flushes, orphans, rejections
  chain_scale       synthetic, SURVEY §9 C2 probe at reduced scale: 300 math_chain_k workflows,
                    log-uniform bases, tight capacity (rejections) and pressure ticks
  *_flaky           alt_pressure / chain_scale with backends whose flush throws (FLAKY below)
  mapped_*_reroute  one-bit / threshold stage mapping under overload (reroute_on_overload)
Synthetic inputs are written to tests/golden/inputs/ and committed with the streams.

Full-scale compact goldens (`python tests/golden/make_golden.py c2_probe c4_probe`, written to
tests/golden/full/, match records WITHOUT token ids — P, M, every op, signal, tick, the action log
and the end counters): the inputs regenerate from the seeded generators below, and the token
streams are re-recorded on the GPU box by the same reference driver (--tok-out) whose compact
projection must equal the committed golden before the GPU replays them.
  c2_probe          SURVEY §9 C2 probe, full size: 10k workflows, 50k requests, 110k signals,
                    sum P = 163,183,335, sum M = 125,426,668
  c4_probe          SURVEY §9 C4 probe 2, full size: 24 x 131,072-token A/B alternating workflows
"""
from __future__ import annotations

import gzip
import json
import math
import os
import random
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/proj"
DRIVER = os.path.join(REPO, "oracle", "_ref", "sf_ref_replay")
INPUTS = os.path.join(HERE, "inputs")  # configs are committed; traces regenerate (seeded)


def sim_backend(ref, model, tier, capacity, maxc, prefill, decode, rule):
    return {"ref": ref, "kind": "simulated", "model": model, "tier": tier,
            "price": {"input_per_1m": 0.1, "output_per_1m": 0.4},
            "sim": {"prefill_ms_per_token": prefill, "decode_ms_per_token": decode,
                    "max_concurrency": maxc, "cache_capacity_tokens": capacity, "output": rule}}


def alt_pressure():
    base = 2048
    rnd = random.Random(0x0A1A + 4)
    stages = []
    for i in range(1, 5):
        stages.append({"id": f"s{i}", "backend": "A" if i % 2 else "B", "model": "m",
                       "prompt_from_payload": f"p{i}", "max_tokens": 16})
    cfg = {
        "label": "alt-pressure",
        "backends": [sim_backend("A", "m", "heavy", 19312, 4, 0.05, 1.0,
                                 {"rule": "constant", "tokens": 0}),
                     sim_backend("B", "m", "heavy", 19312, 4, 0.05, 1.0,
                                 {"rule": "constant", "tokens": 0})],
        "mapper": {"type": "explicit"},
        "memory": {"chain": ["preserve_small_increment"], "tau": 512, "tau_pressure": 0.85,
                   "monitor_interval_ms": 100},
        "workflows": [{"name": "alt", "stages": stages,
                       "dependencies": [["s2", "s1"], ["s3", "s2"], ["s4", "s3"]]}],
    }
    trace = []
    for w in range(24):
        words = [f"a{w}x{rnd.randrange(1 << 20)}" for _ in range(base)]
        payload = {}
        for i in range(1, 5):
            extra = [f"e{w}s{i}x{j}" for j in range(10 * (i - 1))]
            payload[f"p{i}"] = " ".join(words + extra)
        trace.append({"template": "alt", "arrival_ms": 300 * w, "payload": payload})
    return cfg, trace


def chain_scale():
    rnd = random.Random(0x0A1A + 2)
    cfg = {
        "label": "chain-scale",
        "backends": [sim_backend("heavy", "sim-heavy-8b", "heavy", 60000, 16, 0.5, 1.0,
                                 {"rule": "constant", "tokens": 0})],
        "mapper": {"type": "explicit"},
        "memory": {"chain": ["preserve_small_increment", "flush_at_boundary"], "tau": 512,
                   "tau_pressure": 0.85, "monitor_interval_ms": 100},
        "templates": {"math_chain_k": {"backend": "heavy", "k": 5, "append_tokens": 40,
                                       "max_tokens": 64}},
    }
    trace = []
    for w in range(300):
        base = int(math.exp(rnd.uniform(math.log(64), math.log(1024))))
        trace.append({"template": "math_chain_k", "arrival_ms": 5 * w,
                      "payload": {"base_tokens": base}})
    return cfg, trace


def c2_probe():
    """SURVEY §9 C2-scale probe at FULL size: 10,000 math_chain_k workflows (k = 5, base
    log-uniform in [512, 8192] drawn with Python random.seed(2), +256 tokens per stage), arrivals
    every 5 ms, one backend (max_concurrency 64, capacity 1,310,720 tokens), default chain.
    sum P = 163,183,335."""
    random.seed(2)
    bases = [int(math.exp(random.uniform(math.log(512), math.log(8192)))) for _ in range(10_000)]
    cfg = {
        "label": "c2-probe",
        "backends": [sim_backend("heavy", "sim-heavy-8b", "heavy", 1_310_720, 64, 0.05, 1.0,
                                 {"rule": "constant", "tokens": 0})],
        "mapper": {"type": "explicit"},
        "memory": {"chain": ["preserve_small_increment", "flush_at_boundary"], "tau": 512,
                   "tau_pressure": 0.85, "monitor_interval_ms": 100},
        "templates": {"math_chain_k": {"backend": "heavy", "k": 5, "append_tokens": 256,
                                       "max_tokens": 64}},
    }
    trace = [{"template": "math_chain_k", "arrival_ms": 5 * w, "payload": {"base_tokens": b}}
             for w, b in enumerate(bases)]
    return cfg, trace


def c4_probe():
    """SURVEY §9 C4 probe 2 at full size: 24 workflows s1@A -> s2@B -> s3@A -> s4@B, each stage
    prompt the workflow's own distinct 131,072-token text, chain [preserve_small_increment],
    arrivals every 300 ms, both backends at the C4 pool's logical capacity of 1,235,952 tokens
    (77,247 blocks x 16), prefill 0.0095 ms/token. The reference gives: first pressure flush at
    ts 3800 (alt-5@A), 54 flush_under_pressure, 22 capacity rejections on B, end occupancy
    8 / 9 orphaned 128k pins (SURVEY §9 quotes 56 pressure flushes for its unstated timing)."""
    base = 131_072
    rnd = random.Random(0x0A1A + 4)
    stages = []
    for i in range(1, 5):
        stages.append({"id": f"s{i}", "backend": "A" if i % 2 else "B", "model": "m",
                       "prompt_from_payload": "p", "max_tokens": 16})
    cap = 1_235_952
    cfg = {
        "label": "c4-probe",
        "backends": [sim_backend("A", "m", "heavy", cap, 4, 0.0095, 1.0,
                                 {"rule": "constant", "tokens": 0}),
                     sim_backend("B", "m", "heavy", cap, 4, 0.0095, 1.0,
                                 {"rule": "constant", "tokens": 0})],
        "mapper": {"type": "explicit"},
        "memory": {"chain": ["preserve_small_increment"], "tau": 512, "tau_pressure": 0.85,
                   "monitor_interval_ms": 100},
        "workflows": [{"name": "alt", "stages": stages,
                       "dependencies": [["s2", "s1"], ["s3", "s2"], ["s4", "s3"]]}],
    }
    trace = []
    for w in range(24):
        words = " ".join(f"a{w}x{rnd.randrange(1 << 20)}" for _ in range(base))
        trace.append({"template": "alt", "arrival_ms": 300 * w, "payload": {"p": words}})
    return cfg, trace


def mixed_workload_trace(n=24, words=20, lengths=None):
    """proj/traces/mixed_workload.jsonl restated: n single_shot_patch requests at t = 0,
    "repair request i: ctx{i}w0 .. ctx{i}w{words-1}", complexity labels simple for i in [0, 5) and
    [12, 17), complex otherwise, 40 expected output tokens (lengths: per-request word counts)."""
    trace = []
    for i in range(n):
        k = words if lengths is None else lengths[i]
        prompt = f"repair request {i}: " + " ".join(f"ctx{i}w{j}" for j in range(k))
        cx = "simple" if (i < 5 or 12 <= i < 17) else "complex"
        trace.append({"template": "single_shot_patch", "arrival_ms": 0,
                      "payload": {"prompt": prompt, "complexity": cx, "expected_output_tokens": 40}})
    return trace


def one_bit_config(reroute=None, maxc=8):
    """proj/configs/mapped_one_bit.json restated (one-bit routing, the light backend's echo script
    as the classifier)."""
    cfg = {
        "label": "mapped-one-bit",
        "backends": [
            {"ref": "light", "kind": "simulated", "model": "sim-light-4b", "tier": "light",
             "price": {"input_per_1m": 0.1, "output_per_1m": 0.4},
             "sim": {"prefill_ms_per_token": 1.0, "decode_ms_per_token": 10.0, "max_concurrency": maxc,
                     "cache_capacity_tokens": 1000000, "output": {"rule": "script", "name": "one_bit_light"}}},
            {"ref": "heavy", "kind": "simulated", "model": "sim-heavy-8b", "tier": "heavy",
             "price": {"input_per_1m": 0.5, "output_per_1m": 1.5},
             "sim": {"prefill_ms_per_token": 2.0, "decode_ms_per_token": 20.0, "max_concurrency": maxc,
                     "cache_capacity_tokens": 1000000,
                     "output": {"rule": "from_trace", "key": "expected_output_tokens", "fallback_tokens": 40}}}],
        "mapper": {"type": "one_bit", "classifier": "light", "light": "light", "heavy": "heavy"},
        "templates": {"single_shot_patch": {"backend": "heavy", "max_tokens": 4096}},
    }
    if reroute:
        cfg["reroute"] = reroute
    return cfg


REROUTE = {"limit": 3, "alternates": {"heavy": ["light"], "light": ["heavy"]}}


def mapped_one_bit():
    return one_bit_config(), mixed_workload_trace()


def mapped_one_bit_reroute():
    """One-bit routing under overload: max_concurrency 2 and queue limit 3, so the burst of 24
    requests spills onto the alternate backend (reroute_on_overload, orchestrator.cpp:78-87)."""
    return one_bit_config(REROUTE, maxc=2), mixed_workload_trace()


def mapped_threshold_reroute():
    """Threshold routing (score = count_context_tokens, config.cpp:193; light iff score <= 40,
    ties light) over prompts of 4..66 words, with overload rerouting."""
    cfg = one_bit_config(REROUTE, maxc=2)
    cfg["label"] = "mapped-threshold"
    cfg["mapper"] = {"type": "threshold", "threshold": 40, "light": "light", "heavy": "heavy"}
    lengths = [4 + (i * 37) % 63 for i in range(24)]
    lengths[3] = 37  # 40 tokens exactly: the tie goes light (mapper.cpp:30)
    return cfg, mixed_workload_trace(lengths=lengths)


ROUTER_SCENARIOS = {"mapped_one_bit_reroute": mapped_one_bit_reroute,
                    "mapped_threshold_reroute": mapped_threshold_reroute}

FULL = os.path.join(HERE, "full")  # compact full-scale goldens (no token ids)
FULL_SCENARIOS = {"c2_probe": c2_probe, "c4_probe": c4_probe}


def write_inputs(fn, dirpath):
    cfg, trace = fn()
    cp = os.path.join(dirpath, "config.json")
    tp = os.path.join(dirpath, "trace.jsonl")
    with open(cp, "w") as f:
        json.dump(cfg, f)
    with open(tp, "w") as f:
        for rec in trace:
            f.write(json.dumps(rec) + "\n")
    return cp, tp


def compact_line(l):
    """What a compact golden keeps of a stream line (match ops lose their token ids)."""
    return {k: v for k, v in l.items() if k not in ("tok", "toff")}


def run_full(name):
    import tempfile
    os.makedirs(FULL, exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        cp, tp = write_inputs(FULL_SCENARIOS[name], td)
        out = os.path.join(td, "o.jsonl")
        subprocess.run([DRIVER, "--config", cp, "--trace", tp, "--out", out, "--no-tok"], check=True)
        with open(out, "rb") as f, gzip.open(os.path.join(FULL, f"{name}.jsonl.gz"), "wb", 9) as g:
            g.write(f.read())
        n = sum(1 for _ in open(out))
    print(f"{name}: {n} records (compact)")


# Failure-path scenarios: the same inputs with test backends whose flush throws (the drivers'
# --flaky REF:MODE; mode 1 = the first attempt of every flush fails and the retry succeeds, mode
# 2 = every attempt fails, so apply_action gives up and the entry is only unpreserved,
# memory.cpp:189-203, 319-325).
FLAKY = {"alt_pressure_flaky": ("alt_pressure", "A:1,B:2"),
         "chain_scale_flaky": ("chain_scale", "heavy:2")}


def run(name, config_path, trace_path, flaky=None):
    out = os.path.join("/tmp", f"golden_{name}.jsonl")
    subprocess.run([DRIVER, "--config", config_path, "--trace", trace_path, "--out", out] +
                   (["--flaky", flaky] if flaky else []), check=True)
    with open(out, "rb") as f, gzip.open(os.path.join(HERE, f"{name}.jsonl.gz"), "wb", 9) as g:
        g.write(f.read())
    n = sum(1 for _ in open(out))
    print(f"{name}: {n} records")


def main():
    if not os.path.exists(DRIVER):
        sys.exit("build the reference replay driver first: make -C oracle ref")
    os.makedirs(INPUTS, exist_ok=True)
    run("support_demo", f"{REF}/configs/support_demo.json", f"{REF}/traces/support_demo.jsonl")
    run("chain_preserve", f"{REF}/configs/chain_preserve.json", f"{REF}/traces/math_chain.jsonl")
    run("chain_flush", f"{REF}/configs/chain_flush.json", f"{REF}/traces/math_chain.jsonl")
    run("mapped_one_bit", f"{REF}/configs/mapped_one_bit.json", f"{REF}/traces/mixed_workload.jsonl")
    run("single_heavy", f"{REF}/configs/single_heavy.json", f"{REF}/traces/mixed_workload.jsonl")
    for name, fn in (("alt_pressure", alt_pressure), ("chain_scale", chain_scale)):
        cfg, trace = fn()
        cp = os.path.join(INPUTS, f"{name}.config.json")
        tp = os.path.join(INPUTS, f"{name}.trace.jsonl")
        with open(cp, "w") as f:
            json.dump(cfg, f, indent=1)
        with open(tp, "w") as f:
            for rec in trace:
                f.write(json.dumps(rec) + "\n")
        run(name, cp, tp)
    for name, fn in ROUTER_SCENARIOS.items():
        cfg, trace = fn()
        cp = os.path.join(INPUTS, f"{name}.config.json")
        tp = os.path.join(INPUTS, f"{name}.trace.jsonl")
        with open(cp, "w") as f:
            json.dump(cfg, f, indent=1)
        with open(tp, "w") as f:
            for rec in trace:
                f.write(json.dumps(rec) + "\n")
        run(name, cp, tp)
    for name, (base, flaky) in FLAKY.items():
        run(name, os.path.join(INPUTS, f"{base}.config.json"), os.path.join(INPUTS, f"{base}.trace.jsonl"),
            flaky)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # e.g. make_golden.py c2_probe c4_probe (full-scale compact goldens)
        for name in sys.argv[1:]:
            run_full(name)
    else:
        main()
