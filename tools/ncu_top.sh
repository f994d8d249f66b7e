#!/bin/bash
# ncu --set full of one kernel class of the C3 solve (run under gpurun; one ncu per call):
#   tools/ncu_top.sh <tag> <demangled-name regex> <launches to skip> [profile_c3.py args]
# The plain run of the same command must exit 0 first (B200_PROFILING.md).
set -e
tag=$1; re=$2; skip=$3; shift 3
python tools/profile_c3.py "$@" > gpurun_out/${tag}_plain.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -s $skip -c 2 \
    -o gpurun_out/${tag} python tools/profile_c3.py "$@" > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
