#!/bin/bash
# Profiling recipe on the GPU box (run under gpurun from the repo root).
#   tools/prof.sh <tag> <tiles> [kernel regex] [extra bench args...]
# 1) launch list (durations) of the timed steps, 2) one --set full capture of
# the named kernels; both restricted to the timed region (GF_PROFILE_TIMED).
set -u
tag=$1; tiles=$2; kre=${3:-"k_contacts_ss|k_integrate"}; shift 3 || true
mkdir -p gpurun_out
B="python bench.py --tiles $tiles --steps 8 --warmup 4 --no-cpu --no-f64 --e2e-steps 0 --amortised-steps 0 --prof-steps 4 $*"
GF_PROFILE_TIMED=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/launches_$tag.csv $B > gpurun_out/launches_$tag.log 2>&1
python profiles/launch_summary.py gpurun_out/launches_$tag.csv > gpurun_out/launch_summary_$tag.txt 2>&1
GF_PROFILE_TIMED=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k "regex:$kre" -c 4 -f -o gpurun_out/ncu_$tag $B > gpurun_out/ncu_$tag.log 2>&1
ncu -i gpurun_out/ncu_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_raw.csv 2>/dev/null
echo done
