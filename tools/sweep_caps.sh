#!/bin/bash
# Register-cap x CTA-size sweep of the two-sweep marching passes on the GPU box (run under gpurun):
#   tools/sweep_caps.sh <tag> "<cap>:<wpc>[,<wpc>...][:<extra nvcc flags>]" ...
# Rebuilds libpdmg_b200.so per spec (-DPDMG_M2_MAXNREG=<cap> <extra>) and runs one C3 bench per CTA size (PDMG_M2_WPC).
set -u
tag=$1; shift
i=0
for spec in "$@"; do
  IFS=: read -r cap wpcs extra <<< "$spec"
  make -C paper_2203_11154_b200/csrc -B -j16 EXTRA_NVFLAGS="-DPDMG_M2_MAXNREG=$cap ${extra:-}" > gpurun_out/${tag}_v${i}_build.log 2>&1 || { echo "build $spec failed"; tail -5 gpurun_out/${tag}_v${i}_build.log; continue; }
  for w in ${wpcs//,/ }; do
    PDMG_M2_WPC=$w python bench.py --config ${BENCH_CONFIG:-c3} --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_v${i}_w${w}.json 2> gpurun_out/${tag}_v${i}_w${w}.err
    echo "== $spec wpc=$w"
    python tools/bench_summary.py gpurun_out/${tag}_v${i}_w${w}.json > gpurun_out/${tag}_v${i}_w${w}.txt; sed -n 1,8p gpurun_out/${tag}_v${i}_w${w}.txt
  done
  i=$((i+1))
done
