#!/bin/bash
# Profiling recipe for one round (run under gpurun from the repo root; one GPU, never multi-rank):
#   bash profiles/capture.sh <tag>
# Outputs into gpurun_out/<tag>/: the bench line, the launch list of a short bench run and full
# ncu captures of the kernels DESIGN.md reports on (summarised by profiles/ncu_summary.py).
set -u
T=${1:-round}
O=gpurun_out/$T
mkdir -p $O
python bench.py > $O/bench.log 2>&1
tail -1 $O/bench.log > $O/bench_line.json
B="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-c1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > /dev/null 2>&1
F="ncu --set full --clock-control none --import-source on"
Q="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-kv --no-c4 --no-c1"
# C2 step kernels: the 7th match_block / match_chain launch of this command is a timed C2 step;
# the C5 lookup is the 3rd lookup_req launch (one-pass lookup: gate, warm-up, timed)
$F -k regex:match_prep --launch-skip 6 --launch-count 1 -o $O/match_prep $Q > /dev/null 2>&1
$F -k regex:match_block --launch-skip 6 --launch-count 1 -o $O/match_block $Q > /dev/null 2>&1
$F -k regex:match_chain --launch-skip 6 --launch-count 1 -o $O/match_chain $Q > /dev/null 2>&1
$F -k regex:lookup_req --launch-skip 2 --launch-count 1 -o $O/c5_lookup_req $Q > /dev/null 2>&1
$F -k regex:press1 --launch-skip 2 --launch-count 1 -o $O/press1 $Q > /dev/null 2>&1
$F -k regex:chunk_emit --launch-skip 1 --launch-count 1 -o $O/chunk_emit $Q > /dev/null 2>&1
$F -k regex:sig_resolve --launch-skip 1 --launch-count 1 -o $O/sig_resolve $Q > /dev/null 2>&1
$F -k regex:latency_kernel --launch-skip 1 --launch-count 1 -o $O/latency $Q > /dev/null 2>&1
$F -k regex:reroute_window --launch-skip 4 --launch-count 1 -o $O/reroute_window $Q > /dev/null 2>&1
# KV legs: the last payload launch of this command is a timed 200-workflow stage commit, the
# last gather launch a timed 32-pin gather
K="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-c5 --no-mm --no-tok --no-lat --no-c1"
$F -k regex:payload_kernel --launch-skip 9 --launch-count 1 -o $O/payload_commit $K > /dev/null 2>&1
$F -k regex:gather_kernel --launch-skip 2 --launch-count 1 -o $O/gather $K > /dev/null 2>&1
for r in $O/*.ncu-rep; do python profiles/ncu_summary.py $r; done > $O/ncu_summaries.txt 2>&1
ls -la $O
