import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
import paper_2603_13605_b200 as pkg
from paper_2603_13605_b200.abi import Config, Pool
n = int(sys.argv[1]); chunk = int(sys.argv[2]); use_dev = int(sys.argv[3])
wl = bench.make_workload(0x0A1A + 2, n)
mpb = int(bench.blocks_of(wl["req_len"]).max()) + 1
nb = int(bench.blocks_of(wl['base']).sum()) + 2 * mpb + 1024
import math
tl = max(10, int(math.ceil(math.log2(2 * nb))) + 1)
api = pkg.api()
g = Pool(api, Config(max_workflows=n, n_blocks=nb, capacity_tokens=1 << 50, max_pin_blocks=mpb, table_log2=tl))
wf = np.arange(n, dtype=np.int32)
for c0 in range(0, n, chunk):
    c1 = min(n, c0 + chunk)
    off = wl["pin_off"][c0:c1 + 1] - wl["pin_off"][c0]
    tok = wl["pin_tok"][wl["pin_off"][c0]:wl["pin_off"][c1]]
    assert g.commit(wf[c0:c1], off, tok).all()
if use_dev:
    d_wf = torch.from_numpy(wf).cuda(); d_off = torch.from_numpy(wl["req_off"]).cuda()
    d_tok = torch.from_numpy(wl["req_tok"].view(np.int32)).cuda(); d_M = torch.zeros(n, dtype=torch.int64, device="cuda")
    api.check("m", api.match_batch_dev(g.h, n, C.c_void_p(d_wf.data_ptr()), C.c_void_p(d_off.data_ptr()), C.c_void_p(d_tok.data_ptr()), int(wl["req_off"][-1]), C.c_void_p(d_M.data_ptr()), None))
    torch.cuda.synchronize(); api.pool_sync(g.h)
    M = d_M.cpu().numpy()
else:
    M = g.match(wf, wl["req_off"], wl["req_tok"])
bad = np.nonzero(M != wl["expect_M"])[0]
print(f"n={n} chunk={chunk} dev={use_dev}: {len(bad)} bad", bad[:8], M[bad[:8]], wl["expect_M"][bad[:8]], wl["base"][bad[:8]])
# pin hash check for a few workflows vs host chain hashes
lib = pkg.load_library()
