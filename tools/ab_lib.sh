#!/bin/bash
# A/B alternative builds of the library on the GPU box (launch lists under ncu):
#   tools/ab_lib.sh <tiles> <tag> lib_a.so lib_b.so ...   (paths relative to the package)
tiles=$1; tag=$2; shift 2
mkdir -p gpurun_out
for lib in "$@"; do
  n=$(basename $lib .so)
  GF_LIB=$PWD/paper_2311_04648_b200/$lib GF_PROFILE_TIMED=1 timeout 900 ncu --profile-from-start off \
    --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_${tag}_$n.csv \
    python bench.py --tiles $tiles --steps 10 --warmup 4 --no-cpu --no-f64 --e2e-steps 0 --amortised-steps 0 \
    --prof-steps 4 > gpurun_out/ab_${tag}_$n.log 2>&1
  echo "== $n"; python profiles/launch_summary.py gpurun_out/ab_${tag}_$n.csv | head -12
done
