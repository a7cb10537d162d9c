cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --no-pipeline --streams 1 --steps 2 --warmup 3 > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"compress_kernel|decompress" -s 144 -c 48 --csv --log-file gpurun_out/launches.csv python bench.py --no-pipeline --streams 1 --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1; echo ncu=$?
