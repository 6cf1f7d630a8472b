# CUPTI timeline of one stage-commit step (bench kv leg shape), kernels with start/end
import sys, os, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch, ctypes as C
import bench
from torch.profiler import profile, ProfilerActivity

class A: pass
args = A(); args.kv_pool_gib = 64; args.kv_workflows = 200; args.kv_append = 40; args.kv_context = 2008; args.kv_staging_gib = 8; args.warmup = 1; args.steps = 1; args.seed = 0x0A1A
import paper_2603_13605_b200 as pkg
api = pkg.api()
dev = 0
torch.cuda.set_device(dev)
stream = torch.cuda.current_stream()
orig = api.commit_batch_dev
events = []
def wrapped(*a):
    return orig(*a)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    out = bench.kv_legs(args, api, dev, stream, 6536.0, 0)
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
# find the last payload_kernel and print kernels around it
idx = [i for i, e in enumerate(evs) if "payload_kernel" in e.name]
last = idx[-1]
# take the window: from the match_prep before it to the rebuild_done after it
lo = max(i for i in range(last) if "match_prep" in evs[i].name)
hi = min([i for i in range(last, len(evs)) if "rebuild_done" in evs[i].name] + [len(evs) - 1])
t0 = evs[lo].time_range.start
for e in evs[lo:hi + 1]:
    print(f"{(e.time_range.start - t0):9.1f} {(e.time_range.end - t0):9.1f} {e.time_range.elapsed_us():8.1f} {e.name[:70]}")
print(out["stage_commit"])
