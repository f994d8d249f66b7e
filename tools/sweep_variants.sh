#!/bin/bash
# Build-and-bench sweep of compile-time kernel variants on the GPU box (run under gpurun):
#   tools/sweep_variants.sh <tag> "<variant flags 1>" "<variant flags 2>" ...
# Each variant rebuilds libpdmg_b200.so with EXTRA_NVFLAGS and runs one C3 bench (per-kernel CUDA-event times
# in the JSON line); outputs land in gpurun_out/<tag>_v<i>.json.  The last variant's build is left in place.
set -u
tag=$1; shift
cfg=${BENCH_CONFIG:-c3}
i=0
for flags in "$@"; do
  make -C paper_2203_11154_b200/csrc -B -j8 EXTRA_NVFLAGS="$flags" > gpurun_out/${tag}_v${i}_build.log 2>&1 || { echo "build $i failed"; tail -5 gpurun_out/${tag}_v${i}_build.log; }
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/${tag}_v${i}.json 2> gpurun_out/${tag}_v${i}.err
  python - "$flags" gpurun_out/${tag}_v${i}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "FAILED", e); sys.exit(0)
k = d.get("kernels", {})
top = sorted(k.items(), key=lambda kv: -kv[1]["ms"])[:6]
print(f"[{sys.argv[1]}] ms/step {d['ms_per_step']:.3f}  " + "  ".join(f"{n}={v['ms']/v['launches']*1e3:.0f}us" for n, v in top))
PY
  i=$((i+1))
done
