"""Full-scale Class A parity: the SURVEY §9 probes at their configuration sizes, against compact
goldens recorded from the UNMODIFIED reference (tests/golden/make_golden.py c2_probe c4_probe;
tests/golden/full/*.jsonl.gz hold every op, signal, tick, the action log and the end counters —
P and M per request, but no token ids).

  c2_probe  BASELINE configs[1] shape: 10,000 math_chain_k workflows, 50,000 requests, 110,000
            lifecycle signals, sum P = 163,183,335, sum M = 125,426,668
  c4_probe  BASELINE configs[3] shape: 24 A/B-alternating workflows of 131,072-token prompts at the
            C4 pool's logical capacity: 54 flush_under_pressure, 22 capacity rejections, orphans

Two GPU paths are checked, each bit-exact:
  1. the drop-in: the reference's own orchestrator + memory manager + harness loop over the B200
     pool (oracle/_ref/sf_gpu_replay, integration/), with the reference MemoryManager and with
     GpuMemoryManager; the pools start small and grow (sfkv_pool_reserve) — 131,072-token pins
     exceed the initial 4,096-token block tables;
  2. batched pools: the token stream is re-recorded here by the reference driver
     (sf_ref_replay --tok-out), its compact projection must equal the committed golden, then it is
     replayed through GPU pools (batched) and through the CPU oracle.
"""
import gzip
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import replay

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden  # noqa: E402

REF_DRIVER = os.path.join(REPO, "oracle", "_ref", "sf_ref_replay")
GPU_DRIVER = os.path.join(REPO, "oracle", "_ref", "sf_gpu_replay")
NAMES = ["c2_probe", "c4_probe"]


def _golden(name):
    with gzip.open(os.path.join(make_golden.FULL, f"{name}.jsonl.gz"), "rt") as f:
        return [json.loads(line) for line in f]


def _inputs(tmp_path, name):
    return make_golden.write_inputs(make_golden.FULL_SCENARIOS[name], str(tmp_path))


def test_full_goldens_are_the_survey_probes():
    """The committed compact goldens carry the SURVEY §9 totals (CPU: no replay)."""
    g = _golden("c2_probe")
    m = [l for l in g if l.get("op") == "match"]
    assert len(m) == 50_000
    assert sum(l["P"] for l in m) == 163_183_335 and sum(l["M"] for l in m) == 125_426_668
    assert sum(1 for l in g if l["type"] == "sig") == 110_000
    g4 = _golden("c4_probe")
    acts = [l for l in g4 if l["type"] == "act"]
    assert sum(1 for a in acts if a["reason"] == "flush_under_pressure") == 54
    end = g4[-1]["backends"]
    assert end["B"]["capacity_rejections"] == 22
    assert end["A"]["occupancy_tokens"] == 8 * 131_072 and end["B"]["occupancy_tokens"] == 9 * 131_072


def _compare_dropin(got, gold):
    want_req = [(l["b"], l["wf"], l["stage"], l["P"], l["M"]) for l in gold if l.get("op") == "match"]
    got_req = [(l["b"], l["wf"], l["stage"], l["P"], l["M"]) for l in got if l["type"] == "req"]
    assert len(got_req) == len(want_req)
    first_bad = next((i for i, (a, b) in enumerate(zip(got_req, want_req)) if a != b), None)
    assert first_bad is None, (first_bad, got_req[first_bad], want_req[first_bad])
    keys = ("trigger", "ts", "action", "workflow", "backend", "reason")
    want_act = [tuple(l[k] for k in keys) for l in gold if l["type"] == "act"]
    got_act = [tuple(l[k] for k in keys) for l in got if l["type"] == "act"]
    assert got_act == want_act
    gend = next(l for l in gold if l["type"] == "end")
    oend = next(l for l in got if l["type"] == "end")
    assert oend["now_ms"] == gend["now_ms"]
    for ref, want in gend["backends"].items():
        assert oend["backends"][ref] == want, ref


@pytest.mark.gpu
@pytest.mark.parametrize("gpu_memory", [False, True], ids=["ref-memory", "gpu-memory"])
@pytest.mark.parametrize("name", NAMES)
def test_full_scale_dropin_matches_reference(tmp_path, name, gpu_memory):
    if not os.path.exists(GPU_DRIVER):
        pytest.fail("oracle/_ref/sf_gpu_replay missing: build it where /root/reference exists")
    cp, tp = _inputs(tmp_path, name)
    op = os.path.join(str(tmp_path), "o.jsonl")
    subprocess.run([GPU_DRIVER, "--config", cp, "--trace", tp, "--out", op] +
                   (["--gpu-memory"] if gpu_memory else []), check=True, timeout=1200)
    with open(op) as f:
        got = [json.loads(line) for line in f]
    _compare_dropin(got, _golden(name))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_full_scale_batched_pools_match_reference(tmp_path, gpu_api, oracle_api, name):
    if not os.path.exists(REF_DRIVER):
        pytest.fail("oracle/_ref/sf_ref_replay missing: build it where /root/reference exists")
    cp, tp = _inputs(tmp_path, name)
    op, tk = os.path.join(str(tmp_path), "o.jsonl"), os.path.join(str(tmp_path), "tok.u32")
    subprocess.run([REF_DRIVER, "--config", cp, "--trace", tp, "--out", op, "--tok-out", tk],
                   check=True, timeout=1200)
    with open(op) as f:
        stream = [json.loads(line) for line in f]
    assert [make_golden.compact_line(l) for l in stream] == _golden(name), \
        "the re-recorded reference stream differs from the committed golden"
    tokens = np.fromfile(tk, dtype=np.uint32)
    assert replay.replay(stream, gpu_api, batched=True, tokens=tokens) > 0
    if name == "c4_probe":  # and the CPU oracle at full C4 size
        assert replay.replay([dict(l) for l in stream], oracle_api, batched=True, tokens=tokens) > 0


@pytest.mark.gpu
def test_c5_lookup_hit_sets_at_config_scale(gpu_api, oracle_api):
    """BASELINE configs[4] at full size: 1,048,576 resident blocks (8,192 64-way shared system
    prompts + 32,768 private contexts), 100k batched stage-prefix lookups (~9.6 M blocks): every
    out_block id and every hit length equals the CPU oracle's (sfo_lookup_batch), and the hit
    lengths equal the construction's."""
    import bench
    from paper_2603_13605_b200.abi import Pool
    cfg, resident, (off, tok, expect_hit) = bench.c5_workload(0x0A1A + 5, 100_000)
    g, o = Pool(gpu_api, cfg), Pool(oracle_api, cfg)
    for wf, woff, wtok in resident:
        np.testing.assert_array_equal(g.commit(wf, woff, wtok), o.commit(wf, woff, wtok))
    assert g.stats()["table_live"] == o.stats()["table_live"] == 1_048_576
    bg, hg = g.lookup(off, tok)
    bo, ho = o.lookup(off, tok)
    np.testing.assert_array_equal(hg, expect_hit)
    np.testing.assert_array_equal(hg, ho)
    np.testing.assert_array_equal(bg, bo)
    assert (bg >= 0).sum() == int(expect_hit.sum() // 16)
