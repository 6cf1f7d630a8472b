import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, oracle_lib
import paper_2603_13605_b200 as pkg
from paper_2603_13605_b200.abi import Config, Pool
from scenarios import Workload
n_wf = 96
wl = Workload(1, n_wf, n_sys=3, sys_len=(16, 80), ctx_len=(0, 70), append=(0, 50))
cfg = Config(max_workflows=n_wf, n_blocks=6000, capacity_tokens=60_000, max_pin_blocks=64, table_log2=14)
g, o = Pool(pkg.api(), cfg), Pool(oracle_lib.load(), cfg)
rng = np.random.default_rng(101)
wfs = rng.choice(n_wf, size=int(rng.integers(1, n_wf)), replace=False).astype(np.int32)
seqs, off, tok = wl.batch(wfs)
Mg, hg = g.match(wfs, off, tok, want_hash=True)
Mo, ho = o.match(wfs, off, tok, want_hash=True)
nb = (np.diff(off) + 15) // 16
boff = np.concatenate([[0], np.cumsum(nb)])
bad = np.nonzero(hg != ho)[0]
print("n", len(wfs), "items", len(ho), "tokens", off[-1], "bad", len(bad))
for i in bad[:40]:
    r = np.searchsorted(boff, i, side='right') - 1
    print(f"item {i} tile {i//32} lane {i%32} req {r} k {i-boff[r]} nb {nb[r]} len {off[r+1]-off[r]}")
