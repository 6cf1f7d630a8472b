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
