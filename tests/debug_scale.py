import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, bench, oracle_lib
import paper_2603_13605_b200 as pkg
from paper_2603_13605_b200.abi import Config, Pool
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
wl = bench.make_workload(5, n)
nb = int(bench.blocks_of(wl['base']).sum()) + 2000
cfg = Config(max_workflows=n, n_blocks=nb, capacity_tokens=1 << 50, max_pin_blocks=600, table_log2=22)
o = Pool(oracle_lib.load(), cfg); g = Pool(pkg.api(), cfg)
wf = np.arange(n, dtype=np.int32)
for p in (o, g):
    p.commit(wf, wl['pin_off'], wl['pin_tok'])
bad = [w for w in range(0, n, max(1, n // 50)) if not (g.pin_blocks(w)[1] == o.pin_blocks(w)[1]).all()]
print("pins with wrong hashes:", len(bad), bad[:10])
Mo, ho = o.match(wf, wl['req_off'], wl['req_tok'], want_hash=True)
Mg, hg = g.match(wf, wl['req_off'], wl['req_tok'], want_hash=True)
print("M mismatches:", int((Mo != Mg).sum()), "hash mismatches:", int((ho != hg).sum()), "of", len(ho))
idx = np.nonzero(ho != hg)[0]
if len(idx):
    boff = np.concatenate([[0], np.cumsum(bench.blocks_of(np.diff(wl['req_off'])))])
    r = np.searchsorted(boff, idx[:10], side='right') - 1
    print("first bad blocks:", idx[:10], "req", r, "k", idx[:10] - boff[r], "tile", idx[:10] // 256)
