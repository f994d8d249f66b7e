#!/bin/bash
# ncu --set full of one kernel class of the C3 solve (run under gpurun; one ncu per call):
#   tools/ncu_top.sh <tag> <demangled-name regex> <launches to skip> [profile_c3.py args]
# The plain run of the same command must exit 0 first (B200_PROFILING.md).
set -e
tag=$1; re=$2; skip=$3; shift 3
python tools/profile_c3.py "$@" > gpurun_out/${tag}_plain.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -s $skip -c 1 \
    -o /tmp/${tag} python tools/profile_c3.py "$@" > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
# the report itself stays on the box (tens of MB); its raw metrics and per-instruction source page come back
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${tag}_sass.csv.gz || true
ncu -i /tmp/${tag}.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv || true
