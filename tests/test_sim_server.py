"""SimServer protocol over the pool (§8f-4), mirroring the reference's "sim server round trip:
completions, cache reuse, flush, utilization" (proj/tests/test_http_wire.cpp:160-199): a 100-token
prompt is cold, its 130-token extension reuses the 100 pinned tokens over HTTP, utilization is
130/10000, flushing "w" frees 130 and the next call is cold again.

CPU: the host side (HTTP handler, admission, JSON bodies) over the oracle library as the pool.
GPU (`-m gpu`): the same round trip through the sm_100a pool, tokenizer and latency kernels."""
import json
import urllib.error
import urllib.request

import pytest

from paper_2603_13605_b200.sim_server import GpuSimBackend, GpuSimServer, placeholder_text


def synthetic_prompt(n, salt=""):  # templates.cpp:88-96
    return " ".join("%s%d" % (salt, i) for i in range(n))


def _post(url, obj, raw=None):
    body = raw if raw is not None else json.dumps(obj).encode()
    req = urllib.request.Request(url, data=body, headers={"Content-Type": "application/json"}, method="POST")
    with urllib.request.urlopen(req, timeout=10) as r:
        return r.status, r.read().decode()


def _get(url):
    with urllib.request.urlopen(url, timeout=10) as r:
        return r.status, r.read().decode()


def _round_trip(api):
    be = GpuSimBackend(api, "shim", prefill_ms_per_token=0.01, decode_ms_per_token=0.01, max_concurrency=4,
                       cache_capacity_tokens=10000, output_tokens=5, max_workflows=16, max_pin_blocks=64)
    srv = GpuSimServer(be)
    srv.start()
    try:
        ep = srv.endpoint

        def complete(n):
            req = {"model": "m", "messages": [{"role": "user", "content": synthetic_prompt(n)}],
                   "metadata": {"workflow_id": "w", "stage_id": "s"}}
            code, text = _post(ep + "/v1/chat/completions", req)
            assert code == 200
            return json.loads(text), text

        r1, text1 = complete(100)
        assert r1["usage"]["prompt_tokens"] == 100
        assert r1["usage"]["completion_tokens"] == 5
        assert r1["usage"]["prompt_tokens_details"]["cached_tokens"] == 0
        assert r1["choices"][0]["message"]["content"] == placeholder_text(5)
        assert text1 == json.dumps(r1, sort_keys=True, separators=(",", ":"))  # nlohmann's compact dump
        r2, _ = complete(130)
        assert r2["usage"]["prompt_tokens_details"]["cached_tokens"] == 100  # pinned prefix reused
        u = json.loads(_get(ep + "/sim/utilization")[1])
        assert u == {"utilization": 130 / 10000, "occupancy_tokens": 130, "capacity_tokens": 10000}
        assert json.loads(_post(ep + "/sim/flush", {"workflow_id": "w"})[1]) == {"freed_tokens": 130}
        assert json.loads(_get(ep + "/sim/utilization")[1])["utilization"] == 0.0
        r3, _ = complete(130)
        assert r3["usage"]["prompt_tokens_details"]["cached_tokens"] == 0  # flush-then-cold
        assert json.loads(_post(ep + "/sim/flush", {"workflow_id": "nobody"})[1]) == {"freed_tokens": 0}
        assert json.loads(_post(ep + "/sim/flush", None, raw=b"")[1]) == {"freed_tokens": 130}  # everything
        # an unpinned call (no workflow) neither reuses nor pins
        code, text = _post(ep + "/v1/chat/completions", {"model": "m", "max_tokens": 2,
                                                          "messages": [{"role": "user", "content": "a b c"}]})
        r4 = json.loads(text)
        assert r4["usage"] == {"prompt_tokens": 3, "completion_tokens": 2, "prompt_tokens_details": {"cached_tokens": 0}}
        assert json.loads(_get(ep + "/sim/utilization")[1])["occupancy_tokens"] == 0
        with pytest.raises(urllib.error.HTTPError) as e:
            _post(ep + "/v1/chat/completions", None, raw=b"{not json")
        assert e.value.code == 400
    finally:
        srv.stop()
        be.close()


def test_sim_server_round_trip_host_logic(oracle_api):
    _round_trip(oracle_api)


@pytest.mark.gpu
def test_sim_server_round_trip_gpu(gpu_api):
    _round_trip(gpu_api)


@pytest.mark.gpu
def test_sim_backend_grows_and_recycles_slots_gpu(gpu_api):
    """Nothing is capped (the reference's pins are a std::map): more workflows than slots and longer
    prompts than the block table grow the pool in place; a flushed workflow's slot is reused."""
    be = GpuSimBackend(gpu_api, "shim", prefill_ms_per_token=0.001, decode_ms_per_token=0.001,
                       cache_capacity_tokens=100_000, output_tokens=1, max_workflows=2, max_pin_blocks=2)
    try:
        msg = lambda n, s="": [synthetic_prompt(n, s)]  # noqa: E731
        for w in ("a", "b", "c"):
            assert be.complete(msg(100, w), workflow_id=w)["cached_tokens"] == 0
        assert be.pool.cfg.max_workflows >= 3 and be.pool.cfg.max_pin_blocks >= 7
        assert be.complete(msg(130, "a"), workflow_id="a")["cached_tokens"] == 100
        assert be.complete(msg(130, "c"), workflow_id="c")["cached_tokens"] == 100
        slot_a = be.slots["a"]
        assert be.flush("a") == 130
        assert "a" not in be.slots
        assert be.complete(msg(50, "d"), workflow_id="d")["cached_tokens"] == 0
        assert be.slots["d"] == slot_a  # recycled, and cold: the flushed pin is gone
        assert be.complete(msg(60, "d"), workflow_id="d")["cached_tokens"] == 50
        assert be.utilization()["occupancy_tokens"] == 100 + 130 + 60
        assert be.errors == 0
    finally:
        be.close()
