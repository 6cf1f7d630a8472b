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
Synthetic inputs are written to tests/golden/inputs/ and committed with the streams.
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


def run(name, config_path, trace_path):
    out = os.path.join("/tmp", f"golden_{name}.jsonl")
    subprocess.run([DRIVER, "--config", config_path, "--trace", trace_path, "--out", out],
                   check=True)
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


if __name__ == "__main__":
    main()
