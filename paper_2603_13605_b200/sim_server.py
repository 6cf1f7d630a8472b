"""Wire and on-disk formats over the GPU path.

* `GpuSimServer`: the reference's SimServer (proj/src/sim_server.cpp:27-116, sim_server.hpp:10-33)
  — the same HTTP protocol a serving engine speaks — backed by a B200 pool instead of a
  SimulatedBackend: POST /v1/chat/completions, POST /sim/flush, GET /sim/utilization. The
  backend behind it (`GpuSimBackend`) keeps SimulatedBackend's observable semantics on the wall
  clock (simulated_backend.cpp:20-193): FCFS admission over max_concurrency slots (queue time),
  P = whitespace tokens of the concatenated messages (GPU tokenizer + interner), M = LCP against the
  workflow's pin (sfkv_match_batch), ttft / total / service delay from the batched latency model
  (sfmet_latency_batch), a constant `out0 out1 ...` reply truncated to max_tokens, and the pin
  committed (sfkv_commit_batch) when the service delay has elapsed, before the reply is sent.
* `action_log_jsonl`: MemoryManager::export_action_log's JSONL (memory.cpp:389-401) from the GPU
  tracker's records, byte-identical to the reference's (nlohmann::json's compact dump: sorted
  keys, shortest round-trip doubles).
"""
from __future__ import annotations

import json
import threading
import time
from http.server import BaseHTTPRequestHandler, ThreadingHTTPServer

import numpy as np

from .abi import BLOCK_TOKENS, Api, Config, Interner, Pool, SfkvError, latency_batch


def _dump(obj) -> str:
    """nlohmann::json::dump(): compact, object keys in std::map (sorted) order."""
    return json.dumps(obj, sort_keys=True, separators=(",", ":"), ensure_ascii=False)


def action_log_jsonl(records) -> str:
    """records: iterable of dicts {trigger, ts, action, workflow, backend, reason} in log order."""
    return "".join(_dump({"trigger": r["trigger"], "ts": float(r["ts"]), "action": r["action"],
                          "workflow": r["workflow"], "backend": r["backend"], "reason": r["reason"]}) + "\n"
                   for r in records)


def placeholder_text(n: int) -> str:  # simulated_backend.cpp:9-16
    return " ".join("out%d" % i for i in range(n))


class GpuSimBackend:
    """SimulatedBackend's cache + latency semantics over a GPU pool, on the wall clock.

    Workflow ids map to pool slots; a slot returns to a free list once its workflow has no pin and
    no request in flight (after a flush), and the pool grows in place (sfkv_pool_reserve) when
    the slots or the per-pin block table run out, so — like the reference's std::map of pins —
    nothing here is capped. Physical blocks are sized from the logical capacity the way the
    reference-side binding sizes them (integration/gpu_pinned_backend.cpp blocks_for), so a commit
    that logical admission accepts always finds blocks."""

    def __init__(self, api: Api, model: str, prefill_ms_per_token=1.0, decode_ms_per_token=10.0,
                 fixed_overhead_ms=0.0, max_concurrency=1, cache_capacity_tokens=1_000_000,
                 output_tokens=16, device=0, max_workflows=256, max_pin_blocks=256):
        self.api, self.model, self.device = api, model, device
        self.params = (float(fixed_overhead_ms), float(prefill_ms_per_token), float(decode_ms_per_token))
        self.output_tokens = int(output_tokens)
        self.capacity = int(cache_capacity_tokens)
        nb = self._blocks_for(max_workflows, max_pin_blocks)
        self.pool = Pool(api, Config(max_workflows=max_workflows, n_blocks=nb, capacity_tokens=self.capacity,
                                     max_pin_blocks=max_pin_blocks,
                                     table_log2=int(np.ceil(np.log2(2 * nb))) + 1, device=device))
        self.interner = Interner(api, table_log2=16, arena_bytes=1 << 20, device=device)  # grows on demand
        self.slots: dict[str, int] = {}
        self.free = list(range(max_workflows - 1, -1, -1))
        self.inflight: dict[str, int] = {}
        self.lock = threading.Lock()  # one host thread per pool handle
        self.admission = threading.Semaphore(max_concurrency)  # FCFS slots (simulated_backend.cpp:31-47)
        self.errors = 0  # commits that failed on the device (logged non-pins)

    def _blocks_for(self, slots, pin_blocks):
        return self.capacity // BLOCK_TOKENS + slots + 2 * pin_blocks + 64

    def _slot(self, wf: str) -> int:
        if wf not in self.slots:
            if not self.free:  # grow: twice the slots
                mw = 2 * self.pool.cfg.max_workflows
                old = self.pool.cfg.max_workflows
                self.pool.reserve(max_workflows=mw, n_blocks=self._blocks_for(mw, self.pool.cfg.max_pin_blocks))
                self.free = list(range(mw - 1, old - 1, -1))
            self.slots[wf] = self.free.pop()
        return self.slots[wf]

    def _release_if_idle(self, wf: str):
        """After a flush: the workflow has no pin; with nothing in flight its slot is free (a
        request in flight re-pins at completion, so its slot stays)."""
        if wf in self.slots and not self.inflight.get(wf):
            self.inflight.pop(wf, None)
            self.free.append(self.slots.pop(wf))

    def complete(self, messages, workflow_id="", stage_id="", max_tokens=0):
        t0 = time.monotonic()
        with self.admission:
            queue_ms = (time.monotonic() - t0) * 1e3
            with self.lock:
                off, ids = self.interner.tokenize_growing([[m.encode() for m in messages]])
                P = int(off[-1])
                M = 0
                slot = self._slot(workflow_id) if workflow_id else -1
                wfa = np.array([slot], np.int32)
                if slot >= 0:
                    self.inflight[workflow_id] = self.inflight.get(workflow_id, 0) + 1
                    M = int(self.pool.match(wfa, off, ids)[0])
                O = self.output_tokens if max_tokens <= 0 else min(self.output_tokens, max_tokens)
                ttft, total, service = latency_batch(self.api, [0], [queue_ms], [P], [M], [O],
                                                     [self.params[0]], [self.params[1]], [self.params[2]],
                                                     device=self.device)
            time.sleep(float(service[0]) / 1e3)  # the completion event fires after prefill + decode
            with self.lock:
                if slot >= 0:  # pin_prompt at completion (simulated_backend.cpp:125-127)
                    self.inflight[workflow_id] -= 1
                    need = (P + BLOCK_TOKENS - 1) // BLOCK_TOKENS
                    try:
                        if need > self.pool.cfg.max_pin_blocks:  # a longer prompt than any before
                            mb = max(need, 2 * self.pool.cfg.max_pin_blocks)
                            self.pool.reserve(max_pin_blocks=mb,
                                              n_blocks=self._blocks_for(self.pool.cfg.max_workflows, mb))
                        self.pool.commit(wfa, off, ids)
                    except SfkvError:  # the reference never fails a request on pin_prompt
                        self.errors += 1
        return {"content": placeholder_text(O), "prompt_tokens": P, "completion_tokens": O,
                "cached_tokens": M, "queue_ms": queue_ms, "ttft_ms": float(ttft[0]), "total_ms": float(total[0])}

    def flush(self, workflow_id=None) -> int:
        with self.lock:
            if workflow_id is None:
                freed = self.pool.flush(-1)
                for wf in list(self.slots):
                    self._release_if_idle(wf)
                return freed
            if workflow_id not in self.slots:  # nothing pinned for it: frees nothing
                return 0
            freed = self.pool.flush(self.slots[workflow_id])
            self._release_if_idle(workflow_id)
            return freed

    def utilization(self):
        with self.lock:
            st = self.pool.stats()
        return {"utilization": st["occupancy_tokens"] / self.capacity,
                "occupancy_tokens": st["occupancy_tokens"], "capacity_tokens": self.capacity}

    def close(self):
        self.interner.close()
        self.pool.close()


class GpuSimServer:
    """HTTP shim over a GpuSimBackend (the reference SimServer's protocol)."""

    def __init__(self, backend: GpuSimBackend):
        self.backend = backend
        srv = self

        class Handler(BaseHTTPRequestHandler):
            protocol_version = "HTTP/1.1"

            def log_message(self, *a):  # quiet
                pass

            def _send(self, code, obj):
                body = _dump(obj).encode()
                self.send_response(code)
                self.send_header("Content-Type", "application/json")
                self.send_header("Content-Length", str(len(body)))
                self.end_headers()
                self.wfile.write(body)

            def _body(self):
                n = int(self.headers.get("Content-Length", "0") or 0)
                raw = self.rfile.read(n) if n else b""
                try:
                    return json.loads(raw) if raw else None
                except ValueError:
                    return None

            def do_POST(self):
                parsed = self._body()
                if self.path == "/v1/chat/completions":
                    if not isinstance(parsed, dict) or "messages" not in parsed:
                        return self._send(400, {"error": "malformed request"})
                    msgs = [m.get("content") if isinstance(m.get("content"), str) else "" for m in parsed["messages"]]
                    meta = parsed.get("metadata") if isinstance(parsed.get("metadata"), dict) else {}
                    model = parsed.get("model", srv.backend.model)
                    try:
                        r = srv.backend.complete(msgs, meta.get("workflow_id", ""), meta.get("stage_id", ""),
                                                 int(parsed.get("max_tokens", 0) or 0))
                    except Exception:
                        return self._send(500, {"error": "simulation failure"})
                    return self._send(200, {
                        "object": "chat.completion", "model": model,
                        "choices": [{"index": 0, "finish_reason": "stop",
                                     "message": {"role": "assistant", "content": r["content"]}}],
                        "usage": {"prompt_tokens": r["prompt_tokens"], "completion_tokens": r["completion_tokens"],
                                  "prompt_tokens_details": {"cached_tokens": r["cached_tokens"]}}})
                if self.path == "/sim/flush":
                    wf = parsed.get("workflow_id") if isinstance(parsed, dict) else None
                    return self._send(200, {"freed_tokens": srv.backend.flush(wf)})
                self._send(404, {"error": "not found"})

            def do_GET(self):
                if self.path == "/sim/utilization":
                    return self._send(200, srv.backend.utilization())
                self._send(404, {"error": "not found"})

        self.httpd = ThreadingHTTPServer(("127.0.0.1", 0), Handler)
        self.thread = None

    def start(self) -> int:
        self.thread = threading.Thread(target=self.httpd.serve_forever, daemon=True)
        self.thread.start()
        return self.port

    @property
    def port(self) -> int:
        return self.httpd.server_address[1]

    @property
    def endpoint(self) -> str:
        return "http://127.0.0.1:%d" % self.port

    def stop(self):
        self.httpd.shutdown()
        self.httpd.server_close()
        if self.thread:
            self.thread.join()


__all__ = ["GpuSimBackend", "GpuSimServer", "action_log_jsonl", "placeholder_text"]
