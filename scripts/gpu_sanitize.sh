#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over scripts/sanitize_workload.py.  usage: gpu_sanitize.sh <tag>
cd "$(dirname "$0")/.."
TAG=${1:-san}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool python scripts/sanitize_workload.py > gpurun_out/san_${tool}_$TAG.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_$TAG.log | tail -1)"
done
