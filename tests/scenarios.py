"""Seeded synthetic workloads shared by the parity tests and bench.py.

Token ids are u32. Workflows draw a shared "system prompt" (so blocks dedup across workflows),
then private context, then per-stage appends — the math_chain / customer-support shapes the
reference's templates produce (templates.cpp:125-153), at configurable scale.
"""
from __future__ import annotations

import numpy as np

from paper_2603_13605_b200.abi import BLOCK_TOKENS, csr


def splitmix_tokens(rng: np.random.Generator, n: int, vocab: int = 1 << 30):
    return rng.integers(1, vocab, size=n, dtype=np.uint32)


class Workload:
    """A population of workflows whose stage prompts grow by appends (the tau-sized increments
    preserve_small_increment keeps, memory.cpp:116-125) with occasional rewrites (misses)."""

    def __init__(self, seed, n_wf, n_sys=4, sys_len=(16, 64), ctx_len=(1, 80), append=(0, 40),
                 p_rewrite=0.1, p_trunc=0.1, vocab=1 << 30):
        self.rng = np.random.default_rng(seed)
        r = self.rng
        self.vocab = vocab
        self.sys = [splitmix_tokens(r, int(r.integers(*sys_len)), vocab) for _ in range(n_sys)]
        self.cur = []
        for w in range(n_wf):
            s = self.sys[int(r.integers(0, n_sys))]
            ctx = splitmix_tokens(r, int(r.integers(*ctx_len)), vocab)
            self.cur.append(np.concatenate([s, ctx]).astype(np.uint32))
        self.append = append
        self.p_rewrite, self.p_trunc = p_rewrite, p_trunc

    def next_prompt(self, w):
        r = self.rng
        cur = self.cur[w]
        u = r.random()
        if u < self.p_rewrite and len(cur) > 0:  # change a token in the middle: partial hit
            cur = cur.copy()
            cur[int(r.integers(0, len(cur)))] ^= np.uint32(0x5A5A)
        elif u < self.p_rewrite + self.p_trunc and len(cur) > 1:
            cur = cur[: int(r.integers(0, len(cur)))]
        add = splitmix_tokens(r, int(r.integers(*self.append)), self.vocab)
        nxt = np.concatenate([cur, add]).astype(np.uint32)
        self.cur[w] = nxt
        return nxt

    def batch(self, wfs):
        seqs = [self.next_prompt(w) for w in wfs]
        off, tok = csr(seqs)
        return seqs, off, tok


def max_blocks(seqs):
    return max([(len(s) + BLOCK_TOKENS - 1) // BLOCK_TOKENS for s in seqs] + [1])
