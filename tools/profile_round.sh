#!/bin/bash
# Round profile evidence (run under gpurun on one B200). Writes into gpurun_out/prof/:
#   bench.json        the default bench line (no profiler attached)
#   launches.csv      ncu launch list (gpu__time_duration.sum, cold-cache, serialised) of a short bench run
#   <kernel>.csv      ncu --set full details of one launch of each top kernel inside the c2 sequence
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile off > $OUT/ncu_launch.log 2>&1
for k in k_spmv_cdia k_rebuild_top k_rebuild_deferred k_poly k_level_update k_ls_gram1 k_ls_tsqr; do
  timeout 600 ncu --set full --clock-control none -k regex:$k -s 40 -c 1 -o /tmp/$k \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile off > $OUT/ncu_$k.log 2>&1
  ncu -i /tmp/$k.ncu-rep --page details --csv > $OUT/$k.csv 2>> $OUT/ncu_$k.log
  ncu -i /tmp/$k.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > $OUT/${k}_raw.csv 2>> $OUT/ncu_$k.log
done
# c1 / c3 bench lines and the banded-CSR ring SpMV of c3
timeout 400 python bench.py --config c3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 300 python bench.py --config c1 --no-cpu-baseline > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 600 ncu --set full --clock-control none -k regex:k_spmv_ring -s 20 -c 1 -o /tmp/k_spmv_ring \
  python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --profile off > $OUT/ncu_k_spmv_ring.log 2>&1
ncu -i /tmp/k_spmv_ring.ncu-rep --page details --csv > $OUT/k_spmv_ring.csv 2>> $OUT/ncu_k_spmv_ring.log
ncu -i /tmp/k_spmv_ring.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > $OUT/k_spmv_ring_raw.csv 2>> $OUT/ncu_k_spmv_ring.log
