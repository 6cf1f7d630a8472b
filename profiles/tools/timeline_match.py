# CUPTI timeline of C2 match steps (bench workload), kernels with start/end
import sys, os, math
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch, ctypes as C
import bench
from torch.profiler import profile, ProfilerActivity
import paper_2603_13605_b200 as pkg
from paper_2603_13605_b200.abi import Config, Pool
api = pkg.api(); dev = 0; torch.cuda.set_device(dev); stream = torch.cuda.current_stream()
wl = bench.make_workload(0x0A1A, 10000); n = wl["n"]
mpb = int(bench.blocks_of(wl["req_len"]).max()) + 1
nb = int(bench.blocks_of(wl["base"]).sum()) + 2 * mpb + 1024
tl = max(10, int(math.ceil(math.log2(2 * nb))) + 1)
pool = Pool(api, Config(max_workflows=n, n_blocks=nb, capacity_tokens=1 << 50, max_pin_blocks=mpb, table_log2=tl, device=dev))
wf = np.arange(n, dtype=np.int32)
for c0 in range(0, n, 2000):
    c1 = min(n, c0 + 2000)
    off = wl["pin_off"][c0:c1 + 1] - wl["pin_off"][c0]
    assert pool.commit(wf[c0:c1], off, wl["pin_tok"][wl["pin_off"][c0]:wl["pin_off"][c1]]).all()
api.check("ss", api.pool_set_stream(pool.h, C.c_void_p(stream.cuda_stream)))
d_wf = torch.from_numpy(wf).to(dev); d_off = torch.from_numpy(wl["req_off"]).to(dev)
d_tok = torch.from_numpy(wl["req_tok"].view(np.int32)).to(dev)
d_M = torch.zeros(n, dtype=torch.int64, device=dev)
d_h = torch.zeros(int(bench.blocks_of(wl["req_len"]).sum()), dtype=torch.int64, device=dev)
l2 = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
def step(hash_=True):
    api.check("m", api.match_batch_dev(pool.h, n, C.c_void_p(d_wf.data_ptr()), C.c_void_p(d_off.data_ptr()),
              C.c_void_p(d_tok.data_ptr()), int(wl["req_off"][-1]), C.c_void_p(d_M.data_ptr()),
              C.c_void_p(d_h.data_ptr()) if hash_ else None))
FLUSH = os.environ.get("FLUSH", "write")  # write | writeread (dirty lines written back before the step)
def flush():
    l2.zero_()
    if FLUSH == "writeread":
        l2.view(torch.int64).max()  # reads the buffer: the flush's dirty lines leave L2 now
for _ in range(3):
    flush(); step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        flush(); torch.cuda.synchronize(); step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
preps = [i for i, e in enumerate(evs) if "match_prep" in e.name]
for i in preps:
    t0 = evs[i].time_range.start
    for e in evs[i:i + 3]:
        print(f"{(e.time_range.start - t0):8.1f} {(e.time_range.end - t0):8.1f} {e.time_range.elapsed_us():8.1f} {e.name[:60]}")
    print("--")
