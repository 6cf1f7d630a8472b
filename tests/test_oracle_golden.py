"""The CPU oracle against the reference's own golden streams (Class A pinning of the oracle).

Every stream in tests/golden/ was recorded from the unmodified reference replaying a trace
(tests/golden/make_golden.py). The oracle must reproduce every M, admission, flush, preserve,
utilization, pressure victim and final counter — one op at a time and batched."""
import pytest

import replay


@pytest.mark.parametrize("name", replay.stream_names())
@pytest.mark.parametrize("batched", [False, True])
def test_oracle_replays_reference_stream(oracle_api, name, batched):
    lines = replay.load_stream(name)
    n = replay.replay(lines, oracle_api, batched=batched)
    assert n > 0


def test_restated_reference_fixtures_reproduce_their_goldens(tmp_path):
    """The drop-in scenarios restate reference fixture files as Python data (the reference tree is
    absent on the GPU box): support_demo.json x support_demo.jsonl and mapped_one_bit.json x
    mixed_workload.jsonl. Replayed through the unmodified reference here, each restatement must
    reproduce the golden recorded from the reference's own files, record for record."""
    import json
    import os
    import subprocess

    import pytest

    from dropin_scenarios import SCENARIOS
    drv = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "sf_ref_replay")
    if not os.path.exists(drv):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    for name in ("support_demo", "mapped_one_bit"):
        cfg, trace = SCENARIOS[name]()
        cp, tp, op = tmp_path / f"{name}.c.json", tmp_path / f"{name}.t.jsonl", tmp_path / f"{name}.o.jsonl"
        cp.write_text(json.dumps(cfg))
        tp.write_text("".join(json.dumps(r) + "\n" for r in trace))
        subprocess.run([drv, "--config", str(cp), "--trace", str(tp), "--out", str(op)], check=True)
        got = [json.loads(line) for line in op.read_text().splitlines()]
        want = replay.load_stream(name)
        strip = lambda l: {k: v for k, v in l.items() if k not in ("flaky", "label")}  # noqa: E731
        assert [strip(l) for l in got] == [strip(l) for l in want], name
