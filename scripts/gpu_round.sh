# Round measurement: smoke, full GPU tests, bench (N=1) + reference arm, ncu launch list of one
# bench step, and one --set full capture of the compress and decompress kernels.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 600 python bench.py --no-pipeline --streams 1 --steps 2 --warmup 3 > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"compress_kernel|decompress" -s 144 -c 48 --csv --log-file gpurun_out/launches.csv python bench.py --no-pipeline --streams 1 --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1; echo ncu=$?
python scripts/profile_case.py --shape 64,256,56,56 --ratio 100 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"compress_kernel|decompress" -s 6 -c 2 -o gpurun_out/prof_full python scripts/profile_case.py --shape 64,256,56,56 --ratio 100 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
