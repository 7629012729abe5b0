#!/bin/bash
# One parameterised GPU job (run under gpurun from the repo root):
#   tools/gpu_job.sh tests|bench|both [extra bench args...]
# logs land in gpurun_out/ (merged back by gpurun)
set -u
mkdir -p gpurun_out
what=${1:-both}; shift || true
if [[ $what == tests || $what == both ]]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/tests.log 2>&1
  tail -5 gpurun_out/tests.log
fi
if [[ $what == bench || $what == both ]]; then
  timeout 1200 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"; tail -c 1500 gpurun_out/bench.err; head -c 600 gpurun_out/bench.json; echo
fi
