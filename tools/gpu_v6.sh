#!/bin/bash
# v6 product kernel: GPU tests + A/B kernel timings (run under gpurun)
mkdir -p gpurun_out
if [[ -z $NOTEST ]]; then
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/tests.log 2>&1; tail -3 gpurun_out/tests.log
fi
for v in ${V6S:-1 0}; do
  echo "== DIAGMM_PRODUCT_V6=$v"
  DIAGMM_V6_DEBUG=1 DIAGMM_PRODUCT_V6=$v timeout 600 python tools/bench_kernels.py ${CASES:-0 1 6 7 9 10 11} 2>&1 | sort | uniq | tail -40
done
