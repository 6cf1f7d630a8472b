"""Match-path stress shapes against the CPU oracle (M and chained hashes bit for bit). Written for
the one-launch span pass this round measured and dropped (commit 050696d), they
now exercise the prep / block / chain path on the batch shapes that stress any decomposition:
requests crossing many tiles with the first mismatch in any of them (or at a tile / span
boundary), thousands of tiny and empty requests (tiles crossing dozens of requests, the
request-window fallback of the block pass), batch lengths at exact multiples of 2048 tokens,
successive launches of very different sizes on one pool (the prep look-back statuses are
epoch-tagged in a per-pool buffer, never cleared between launches), repeated and unpinned
workflows. Reference semantics: prefix_match (simulated_backend.cpp:153-162)."""
import numpy as np
import pytest

from paper_2603_13605_b200.abi import Config, Pool, csr

pytestmark = pytest.mark.gpu

SPAN = 2048


def _pools(gpu_api, oracle_api, n_wf, max_pin_blocks):
    cfg = Config(max_workflows=n_wf, n_blocks=max(4096, n_wf * max_pin_blocks + 64), capacity_tokens=1 << 40,
                 max_pin_blocks=max_pin_blocks, table_log2=17)
    return Pool(gpu_api, cfg), Pool(oracle_api, cfg)


def _check(g, o, wfs, seqs):
    off, tok = csr(seqs)
    Mg, hg = g.match(wfs, off, tok, want_hash=True)
    Mo, ho = o.match(wfs, off, tok, want_hash=True)
    np.testing.assert_array_equal(Mg, Mo)
    np.testing.assert_array_equal(hg, ho)
    Mg2 = g.match(wfs, off, tok)  # M only (no hashes): the other kernel instantiation
    np.testing.assert_array_equal(Mg2, Mo)
    return Mo


def _pin(g, o, wfs, seqs):
    off, tok = csr(seqs)
    np.testing.assert_array_equal(g.commit(wfs, off, tok), o.commit(wfs, off, tok))


def _mutate(rng, s, where):
    s = np.array(s, dtype=np.uint32)
    if len(s) and where is not None:
        s[min(where, len(s) - 1)] ^= 0x5A5A
    return s


def test_span_long_requests_mismatch_in_every_span(gpu_api, oracle_api):
    """Requests of 20k-40k tokens cross 10-20 spans; the first mismatch sits in a different span of
    each request (or nowhere), and some requests are shorter / longer than their pin."""
    rng = np.random.default_rng(11)
    n = 24
    g, o = _pools(gpu_api, oracle_api, n, 2600)
    wfs = np.arange(n, dtype=np.int32)
    pins = [rng.integers(1, 1 << 30, size=int(rng.integers(20_000, 40_000))).astype(np.uint32) for _ in range(n)]
    _pin(g, o, wfs, pins)
    seqs = []
    for i, p in enumerate(pins):
        kind = i % 4
        if kind == 0:    # prefix of the pin, mismatch in span i
            s = _mutate(rng, p[: len(p) - 100], (i * SPAN + 37) % (len(p) - 100))
        elif kind == 1:  # the whole pin plus an append (no mismatch)
            s = np.concatenate([p, rng.integers(1, 99, size=int(rng.integers(0, 300))).astype(np.uint32)])
        elif kind == 2:  # mismatch right at a span boundary
            s = _mutate(rng, p, min(len(p) - 1, (i + 3) * SPAN))
        else:            # shorter than the pin, no mismatch
            s = p[: int(rng.integers(1, len(p)))]
        seqs.append(s)
    M = _check(g, o, wfs, seqs)
    assert (M > 0).all()


def test_span_dense_tiny_and_empty_requests(gpu_api, oracle_api):
    """Thousands of 0-20-token requests: tiles that cross dozens of requests (the block pass's
    request-window fallback); empty requests among them and at the batch end."""
    rng = np.random.default_rng(12)
    n = 3000
    g, o = _pools(gpu_api, oracle_api, n, 4)
    wfs = np.arange(n, dtype=np.int32)
    pins = [rng.integers(1, 50, size=int(rng.integers(0, 24))).astype(np.uint32) for _ in range(n)]
    _pin(g, o, wfs[::2], [pins[i] for i in range(0, n, 2)])  # half the workflows hold a pin
    seqs = []
    for i in range(n):
        r = rng.random()
        if r < 0.25:
            seqs.append(np.zeros(0, dtype=np.uint32))
        elif r < 0.6:
            seqs.append(pins[i][: int(rng.integers(0, len(pins[i]) + 1))])
        else:
            seqs.append(_mutate(rng, rng.integers(1, 50, size=int(rng.integers(1, 21))), int(rng.integers(0, 20))))
    seqs[-5:] = [np.zeros(0, dtype=np.uint32)] * 5
    _check(g, o, wfs, seqs)


@pytest.mark.parametrize("tail", [0, 1, 15, 16, 17])
def test_span_exact_multiples_and_boundaries(gpu_api, oracle_api, tail):
    """Batch lengths of k * 2048 + tail tokens; requests that end exactly on a span boundary, that
    start one token before one, and a single request filling whole spans."""
    rng = np.random.default_rng(13 + tail)
    lens = [SPAN, SPAN - 1, 1, SPAN, 3 * SPAN, 16, SPAN - 16, 0, 5 * SPAN + tail]
    n = len(lens)
    g, o = _pools(gpu_api, oracle_api, n, 5 * SPAN // 16 + 8)
    wfs = np.arange(n, dtype=np.int32)
    pins = [rng.integers(1, 1 << 20, size=L + 40).astype(np.uint32) for L in lens]
    _pin(g, o, wfs, pins)
    seqs = [p[:L] for p, L in zip(pins, lens)]
    seqs[4] = _mutate(rng, seqs[4], 2 * SPAN + 5)
    M = _check(g, o, wfs, seqs)
    assert M[0] == SPAN and M[7] == 0
    # a single request alone
    _check(g, o, wfs[:1], [pins[0][: 4 * SPAN - 3] if len(pins[0]) >= 4 * SPAN else pins[8][: 4 * SPAN]])


def test_span_launches_of_alternating_size(gpu_api, oracle_api):
    """Large, small, large, tiny, larger launches in a row on one pool: stale look-back statuses
    left by a larger earlier launch must never be read as current (epoch-tagged prep statuses)."""
    rng = np.random.default_rng(14)
    n = 64
    g, o = _pools(gpu_api, oracle_api, n, 1100)
    wfs = np.arange(n, dtype=np.int32)
    pins = [rng.integers(1, 1 << 16, size=int(rng.integers(100, 17_000))).astype(np.uint32) for _ in range(n)]
    _pin(g, o, wfs, pins)
    for k in (64, 3, 64, 1, 40, 2, 64, 64):
        sel = np.sort(rng.choice(n, size=k, replace=False)).astype(np.int32)
        seqs = [_mutate(rng, pins[w][: int(rng.integers(0, len(pins[w]) + 1))],
                        int(rng.integers(0, 20_000)) if rng.random() < 0.5 else None) for w in sel]
        _check(g, o, sel, seqs)


def test_span_unpinned_and_repeated_workflows(gpu_api, oracle_api):
    """The same workflow several times in one batch, workflows with no pin, and an empty pin."""
    rng = np.random.default_rng(15)
    n = 8
    g, o = _pools(gpu_api, oracle_api, n, 64)
    base = rng.integers(1, 1000, size=900).astype(np.uint32)
    _pin(g, o, np.array([0, 1, 2], dtype=np.int32), [base, base[:300], np.zeros(0, dtype=np.uint32)])
    wfs = np.array([0, 0, 1, 3, 2, 0, 1, 4], dtype=np.int32)
    seqs = [base, base[:500], base, base, base[:10], _mutate(rng, base, 777), base[:299], base[:17]]
    M = _check(g, o, wfs, seqs)
    assert list(M[:3]) == [900, 500, 300] and M[3] == 0 and M[4] == 0
