#!/bin/bash
# One gpurun lease: GPU tests, the default bench line, kernel micro-benchmarks, the column-loop
# timeline and the teacher-forced full-size parity of whatever corpus travelled in parity_data/.
set -u
OUT=gpurun_out/r02
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
timeout 900 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
for c in ${KBENCH:-c2}; do timeout 300 python tools/kbench.py $c > $OUT/kbench_$c.log 2>&1; done
if [ -f paper_1604_06043_b200/libmstab_b200_tl.so ]; then
  timeout 300 python tools/timeline.py c2 30 > $OUT/timeline_c2.json 2> $OUT/timeline_c2.err
fi
for c in ${PARITY:-}; do
  timeout 1800 python tools/parity_fullsize.py $c ${LIVE:-} > $OUT/parity_$c.txt 2> $OUT/parity_$c.err
done
tail -3 $OUT/pytest_gpu.log 2>/dev/null; head -c 600 $OUT/bench_c2.json; cat $OUT/kbench_*.log
