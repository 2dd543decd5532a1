#!/bin/bash
# compute-sanitizer over the kernel-level, solve-level and preconditioner GPU tests (SURVEY.md §5,
# VERDICT r01 item 8): memcheck (global/shared out-of-bounds, misaligned, leaks off), racecheck
# (shared-memory hazards: block_totals / cta_commit staging, the TMA staging buffers and mbarriers of
# k_spmv_ring2, the cp.async prefetch of k_rebuild_top), synccheck (barrier / mbarrier misuse). One
# gpurun lease; summaries land in gpurun_out/sanitize/ and are copied to profiles/ by hand.
set -u
OUT=gpurun_out/sanitize
mkdir -p $OUT
SEL="${SAN_TESTS:-tests/test_gpu_kernels.py tests/test_gpu_solve.py tests/test_gpu_precond.py tests/test_gpu_complex.py}"
for tool in ${SAN_TOOLS:-memcheck racecheck synccheck}; do
  timeout ${SAN_TIMEOUT:-1500} /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    --log-file $OUT/$tool.log python -m pytest $SEL -m gpu -x -q -p no:cacheprovider > $OUT/$tool.pytest.log 2>&1
  echo "$tool rc=$?" >> $OUT/summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $OUT/$tool.log $OUT/$tool.pytest.log | tail -4 >> $OUT/summary.txt
done
cat $OUT/summary.txt
