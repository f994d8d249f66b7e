#!/bin/bash
# Round evidence on the GPU box (run under gpurun): tools/evidence.sh <tag> [skip-tests]
# GPU tests, bench lines of every BASELINE config, the reference arm, the ncu launch list of the default bench
# command and full ncu captures of the two dominant kernels.  Everything lands in gpurun_out/<tag>_*.
set -u
tag=$1
if [ "${2:-}" != "skip-tests" ]; then
  python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${tag}_pytest_gpu.log
fi
python bench.py > gpurun_out/${tag}_bench_c3.json 2> gpurun_out/${tag}_bench_c3.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_reference_arm_c3.json 2>/dev/null
for c in c1 c2 c4a c4b c5; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$c.json 2>/dev/null; done
python bench.py --config c4a --precision c64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_c4a_c64.json 2>/dev/null
for s in 128 64 32; do python bench.py --shifts $s --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_c3_s$s.json 2>/dev/null; done
python tools/bench_summary.py gpurun_out/${tag}_bench_*.json | grep "ms/step"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_launches_ncu.log 2>&1
bash tools/ncu_top.sh ${tag}_restrict 'k_march2<double, \(bool\)1, \(bool\)0, \(int\)2, \(bool\)1, \(bool\)1, \(int\)512>' 3
bash tools/ncu_top.sh ${tag}_prolong 'k_march2<double, \(bool\)1, \(bool\)1, \(int\)0, \(bool\)0, \(bool\)1, \(int\)512>' 3
