#!/bin/bash
# A/B of the working tree's library against the build of the sources staged under build/head (git archive HEAD),
# alternating runs in one gpurun session:  tools/ab_head.sh <tag> [rounds] [bench args]
set -u
tag=$1; rounds=${2:-2}; shift; shift || true
make -C build/head/paper_2203_11154_b200/csrc -j16 > gpurun_out/${tag}_headbuild.log 2>&1 || { echo "head build failed"; tail -5 gpurun_out/${tag}_headbuild.log; exit 1; }
HEADLIB=$PWD/build/head/paper_2203_11154_b200/libpdmg_b200.so
for r in $(seq 1 $rounds); do
  PDMG_B200_LIB=$HEADLIB python bench.py --steps 8 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/${tag}_head_$r.json 2> gpurun_out/${tag}_head_$r.err
  python bench.py --steps 8 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/${tag}_new_$r.json 2> gpurun_out/${tag}_new_$r.err
done
python tools/bench_summary.py gpurun_out/${tag}_head_*.json gpurun_out/${tag}_new_*.json | grep -v "pack\|finalize\|pass+norm\|coarse_tail"
