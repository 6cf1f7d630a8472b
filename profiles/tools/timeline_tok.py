# CUPTI timeline of one steady-state tokenizer batch (bench tokenize leg shape)
import sys, os, ctypes as C
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import bench
from torch.profiler import profile, ProfilerActivity
import paper_2603_13605_b200 as pkg
from paper_2603_13605_b200.abi import Interner
api = pkg.api(); dev = 0; torch.cuda.set_device(dev); stream = torch.cuda.current_stream()
wl = bench.make_workload(0x0A1A, 10000)
text, tbo = bench.render_text(wl["req_tok"])
n = wl["n"]; msg_off = tbo[wl["req_off"]]; req = np.arange(n + 1, dtype=np.int64); nbytes = int(msg_off[-1])
it = Interner(api, table_log2=20, arena_bytes=16 << 20, device=dev)
api.check("ss", api.interner_set_stream(it.h, C.c_void_p(stream.cuda_stream)))
d_req = torch.from_numpy(req).to(dev); d_moff = torch.from_numpy(msg_off).to(dev)
d_text = torch.from_numpy(np.concatenate([text, np.zeros(16, np.uint8)])).to(dev)
d_off = torch.zeros(n + 1, dtype=torch.int64, device=dev); d_tok = torch.zeros((nbytes + n + 1) // 2 + 1, dtype=torch.int32, device=dev)
d_nt = torch.zeros(1, dtype=torch.int64, device=dev)
def step():
    api.check("t", api.tokenize_batch_dev(it.h, n, C.c_void_p(d_req.data_ptr()), n, C.c_void_p(d_moff.data_ptr()),
              C.c_void_p(d_text.data_ptr()), nbytes, C.c_void_p(d_off.data_ptr()), C.c_void_p(d_tok.data_ptr()),
              C.c_void_p(d_nt.data_ptr())))
for _ in range(3): step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step(); torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = evs[0].time_range.start
for e in evs:
    print(f"{(e.time_range.start - t0):8.1f} {(e.time_range.end - t0):8.1f} {e.time_range.elapsed_us():8.1f} {e.name[:60]}")
