#!/bin/bash
# whole-graph ncu capture (concurrency preserved): duration and DRAM bytes of the bench's compress and decompress graph replays
#   bash scripts/gpu_ncu_graph.sh [variant]
mkdir -p gpurun_out
v=${1:-}
lib=paper_2410_12707_b200/_lib/libadatopk.so
[ -n "$v" ] && lib=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so
GP_LIB=$lib GP_BENCH_SPINUP=0 timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum \
  --clock-control none -c 3000 --csv --log-file gpurun_out/graph_${v:-cur}.csv python bench.py --no-pipeline --no-sweep --steps 2 --warmup 3 > gpurun_out/graph_${v:-cur}.log 2>&1
echo "rc=$?"
