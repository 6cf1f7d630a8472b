import csv, sys, subprocess
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
for v in rows[2:]:
    name = v[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    d = {}
    for i, h in enumerate(hdr):
        if 'pcsamp_warps_issue_stalled' in h and 'not_issued' not in h:
            try: d[h] = float(v[i])
            except: pass
    tot = sum(d.values()) or 1
    print("==", name[:80])
    for h in ('gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
              'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
              'launch__registers_per_thread', 'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct'):
        if h in hdr: print(f"   {h} = {v[hdr.index(h)]} {units[hdr.index(h)]}")
    for h, x in sorted(d.items(), key=lambda t: -t[1])[:5]:
        print(f"   {100*x/tot:5.1f}% {h.replace('smsp__pcsamp_warps_issue_stalled_','stall_')}")
