# CUPTI timeline of the e2e call (sfkv_match_batch through the host-pointer ABI): copies + kernels
import sys, os, math, time, ctypes as C
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import bench
from torch.profiler import profile, ProfilerActivity
import paper_2603_13605_b200 as pkg
from paper_2603_13605_b200.abi import Config, Pool
api = pkg.api(); dev = 0; torch.cuda.set_device(dev)
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
h_wf = torch.from_numpy(wf).pin_memory().numpy()
h_off = torch.from_numpy(wl["req_off"]).pin_memory().numpy()
h_tok = torch.from_numpy(wl["req_tok"].view(np.int32)).pin_memory().numpy().view(np.uint32)
h_M = torch.zeros(n, dtype=torch.int64).pin_memory().numpy()
def step():
    api.check("m", api.match_batch(pool.h, n, h_wf.ctypes.data, h_off.ctypes.data, h_tok.ctypes.data, h_M.ctypes.data, None))
for _ in range(3): step()
t0 = time.perf_counter(); step(); print("wall ms", 1e3 * (time.perf_counter() - t0))
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{(e.time_range.start - t0):9.1f} {(e.time_range.end - t0):9.1f} {e.time_range.elapsed_us():9.1f} {e.name[:60]}")
cpu = sorted([e for e in prof.events() if e.device_type.name == "CPU"], key=lambda e: e.time_range.start)
for e in cpu[:12]:
    print("CPU", f"{e.time_range.elapsed_us():9.1f}", e.name[:60])
