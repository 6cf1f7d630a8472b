"""Tokenizer + interner (§8f-2) against the reference's tokenize_whitespace /
context_token_sequence (backend.cpp:60-91).

CPU: the oracle restatement reproduces the reference's token strings for every request of seeded
random texts (all six C-locale space bytes, runs of separators, leading/trailing space, empty and
all-space messages, requests without messages, bytes >= 0x80, tokens longer than 8 bytes) and
numbers new strings in first-occurrence order. GPU (`-m gpu`): the sm_100a tokenizer returns the
same ids as the oracle across several batches through one persistent interner, and a batch that
overflows the interner fails without changing it."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2603_13605_b200.abi import Interner, SfkvError

REF_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "libsfref.so")
SPACES = [b" ", b"\t", b"\n", b"\v", b"\f", b"\r"]


def random_requests(seed, n=40, vocab=300):
    rng = np.random.default_rng(seed)
    words = []
    for i in range(vocab):
        L = int(rng.choice([1, 2, 3, 5, 8, 9, 15, 17, 40]))
        w = bytes(int(x) for x in rng.integers(33, 256, size=L))
        words.append(w.replace(b"\x85", b"#").replace(b"\xa0", b"%"))  # non-space in the C locale anyway
    reqs = []
    for _ in range(n):
        msgs = []
        for _ in range(int(rng.integers(0, 5))):
            parts = [b"".join(SPACES[int(j)] for j in rng.integers(0, 6, size=int(rng.integers(0, 3))))]
            for _ in range(int(rng.integers(0, 30))):
                parts.append(words[int(rng.integers(0, vocab))])
                parts.append(b"".join(SPACES[int(j)] for j in rng.integers(0, 6, size=int(rng.integers(1, 4)))))
            if rng.random() < 0.5:
                parts.pop()  # no trailing separator: the token ends at the message end
            msgs.append(b"".join(parts))
        reqs.append(msgs)
    return reqs


def ref_tokens(L, msgs):
    n = len(msgs)
    arr = (C.c_char_p * max(n, 1))(*msgs)
    lens = (C.c_longlong * max(n, 1))(*[len(m) for m in msgs])
    cap = sum(len(m) for m in msgs) + 1
    out = C.create_string_buffer(cap)
    out_len = (C.c_longlong * cap)()
    k = L.sfref_context_tokens(n, arr, lens, out, cap, out_len, cap)
    assert k >= 0
    toks, o = [], 0
    for i in range(k):
        toks.append(out.raw[o:o + out_len[i]])
        o += out_len[i]
    return toks


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_tokenizer_matches_reference(oracle_api, seed):
    L = C.CDLL(REF_LIB)
    L.sfref_context_tokens.restype = C.c_longlong
    L.sfref_context_tokens.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_longlong), C.c_char_p,
                                       C.c_longlong, C.POINTER(C.c_longlong), C.c_longlong]
    it = Interner(oracle_api, table_log2=14, arena_bytes=1 << 20)
    reqs = random_requests(seed)
    off, tok = it.tokenize(reqs)
    for r, msgs in enumerate(reqs):
        got = [it.token(i) for i in tok[off[r]:off[r + 1]]]
        assert got == ref_tokens(L, msgs), r
    # first-occurrence numbering
    seen = -1
    for i in tok:
        assert i <= seen + 1
        seen = max(seen, int(i))
    assert it.size() == seen + 1


@pytest.mark.gpu
def test_gpu_tokenizer_matches_oracle_across_batches(gpu_api, oracle_api):
    g = Interner(gpu_api, table_log2=14, arena_bytes=1 << 20)
    o = Interner(oracle_api, table_log2=14, arena_bytes=1 << 20)
    for seed in range(5):  # one interner across batches: ids persist, new ones continue
        reqs = random_requests(100 + seed, n=int(30 + 40 * seed))
        go, gt = g.tokenize(reqs)
        oo, ot = o.tokenize(reqs)
        np.testing.assert_array_equal(go, oo)
        np.testing.assert_array_equal(gt, ot)
        assert g.size() == o.size()
    for i in range(0, o.size(), 7):
        assert g.token(i) == o.token(i)
    # empty batch / empty text
    assert g.tokenize([[], [b"   "], [b""]])[1].size == 0


@pytest.mark.gpu
def test_gpu_interner_overflow_fails_without_change(gpu_api):
    g = Interner(gpu_api, table_log2=6, arena_bytes=64)  # 32 ids, 64 arena bytes
    g.tokenize([[b"a b c"]])
    n0 = g.size()
    with pytest.raises(SfkvError):
        g.tokenize([[b" ".join(b"w%03d" % i for i in range(40))]])
    assert g.size() == n0
    off, tok = g.tokenize([[b"c a b d"]])  # still usable, old ids intact
    assert tok.tolist() == [2, 0, 1, 3]


@pytest.mark.gpu
def test_gpu_interner_reserve_keeps_ids(gpu_api, oracle_api):
    """A tiny interner that grows in place whenever a batch does not fit (sfkv_interner_reserve:
    larger table re-indexed by the same keys, arena copied) hands out exactly the ids a large one
    does, batch after batch — short (exact-key) and long (hash + verify) tokens alike."""
    g = Interner(gpu_api, table_log2=5, arena_bytes=32)
    o = Interner(oracle_api, table_log2=20, arena_bytes=16 << 20)
    grown = 0
    for seed in range(6):
        reqs = random_requests(300 + seed, n=int(20 + 30 * seed))
        lg0 = g.arena()[2]
        go, gt = g.tokenize_growing(reqs)
        grown += g.arena()[2] > lg0
        oo, ot = o.tokenize(reqs)
        np.testing.assert_array_equal(go, oo)
        np.testing.assert_array_equal(gt, ot)
        assert g.size() == o.size()
    assert grown >= 3
    for i in range(0, o.size(), 3):
        assert g.token(i) == o.token(i)


def _edge_batches():
    rng = np.random.default_rng(5)
    one_byte = [[bytes([97 + i % 26]) for i in range(5000)], [b"x"] * 3 + [b" "], []]  # 4096 tokens in a chunk
    long_words = []
    for _ in range(6):  # tokens up to 600 bytes: across chunk boundaries and past the staged window
        words = [bytes(int(x) for x in rng.integers(33, 127, size=int(rng.integers(1, 600)))) for _ in range(40)]
        long_words.append([b" ".join(words), b"\t".join(words[:7])])
    return [one_byte, long_words]


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
def test_oracle_tokenizer_edge_batches_match_reference(oracle_api):
    L = C.CDLL(REF_LIB)
    L.sfref_context_tokens.restype = C.c_longlong
    L.sfref_context_tokens.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_longlong), C.c_char_p,
                                       C.c_longlong, C.POINTER(C.c_longlong), C.c_longlong]
    it = Interner(oracle_api, table_log2=16, arena_bytes=1 << 20)
    for reqs in _edge_batches():
        off, tok = it.tokenize(reqs)
        for r, msgs in enumerate(reqs):
            assert [it.token(i) for i in tok[off[r]:off[r + 1]]] == ref_tokens(L, msgs), r


@pytest.mark.gpu
def test_gpu_tokenizer_edge_batches_match_oracle(gpu_api, oracle_api):
    g = Interner(gpu_api, table_log2=16, arena_bytes=1 << 20)
    o = Interner(oracle_api, table_log2=16, arena_bytes=1 << 20)
    for reqs in _edge_batches():
        go, gt = g.tokenize(reqs)
        oo, ot = o.tokenize(reqs)
        np.testing.assert_array_equal(go, oo)
        np.testing.assert_array_equal(gt, ot)
    assert g.size() == o.size()


@pytest.mark.gpu
def test_gpu_cold_batch_and_reset(gpu_api, oracle_api):
    """A batch of only new strings (the cold path: every token pending, owners ranked by a
    (count, bytes) tile scan, arena written through shared memory or, for tiles of long strings,
    byte by byte) gives the oracle's ids and arena bytes; sfkv_interner_reset empties the
    interner, after which the same batch gets the same ids again."""
    rng = np.random.default_rng(77)
    words = [b"w%07d" % i + bytes(int(x) for x in rng.integers(97, 123, size=int(rng.integers(0, 17))))
             for i in range(20_000)]
    words += [bytes(int(x) for x in rng.integers(33, 127, size=int(rng.integers(50, 300)))) for _ in range(300)]
    reqs = [[b" ".join(words[i:i + 500])] for i in range(0, len(words), 500)]
    g = Interner(gpu_api, table_log2=16, arena_bytes=4 << 20)
    for rep in range(2):
        o = Interner(oracle_api, table_log2=16, arena_bytes=4 << 20)
        go, gt = g.tokenize(reqs)
        oo, ot = o.tokenize(reqs)
        np.testing.assert_array_equal(go, oo)
        np.testing.assert_array_equal(gt, ot)
        assert g.size() == o.size() == len(set(words))
        for i in list(range(0, 50)) + list(range(o.size() - 350, o.size(), 7)):
            assert g.token(i) == o.token(i)
        g.reset()
        assert g.size() == 0


def _boundary_batch(total, seed):
    """Two requests whose text is exactly `total` bytes in all (one message per piece): random
    words over all six C-locale spaces, message starts in the middle of words."""
    rng = np.random.default_rng(seed)
    spaces = b" \t\n\v\f\r"
    raw = bytearray(rng.integers(33, 127, size=total).astype(np.uint8).tobytes())
    for i in rng.choice(total, size=total // 5, replace=False):
        raw[i] = spaces[int(rng.integers(0, 6))]
    cuts = sorted(set(int(c) for c in rng.integers(1, max(2, total), size=6)))
    pieces, prev = [], 0
    for c in cuts + [total]:
        if c > prev:
            pieces.append(bytes(raw[prev:c]))
            prev = c
    h = max(1, len(pieces) // 2)  # two requests; the batch's text is exactly `total` bytes
    return [pieces[:h], pieces[h:]]


@pytest.mark.gpu
@pytest.mark.parametrize("total", [2047, 2048, 2049, 2048 + 255, 2048 + 256, 2048 + 257, 4095, 4096, 4097,
                                   4096 + 256, 6144 + 1])
def test_gpu_tokenizer_chunk_boundaries_match_oracle(gpu_api, oracle_api, total):
    """Texts ending at and around the 2 KiB chunk and the chunk + 256-byte staged window: the count
    pass's full-chunk fast path and the emit pass's full-window fast path against their generic
    paths (the text's last chunks), message starts inside words, every C-locale space."""
    g = Interner(gpu_api, table_log2=16, arena_bytes=1 << 20)
    o = Interner(oracle_api, table_log2=16, arena_bytes=1 << 20)
    for seed in range(3):
        reqs = _boundary_batch(total, seed)
        go, gt = g.tokenize(reqs)
        oo, ot = o.tokenize(reqs)
        np.testing.assert_array_equal(go, oo)
        np.testing.assert_array_equal(gt, ot)
    assert g.size() == o.size()
