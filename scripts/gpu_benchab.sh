# bench (no pipeline) for the default build and each variant; parity tests first
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/gpu_tests.log
for v in default paper_2410_12707_b200/_lib/variants/*/; do
[ $v = default ] || [ -d "$v" ] || continue
n=$(basename $v)
if [ $v = default ]; then L=""; else L=$v/libadatopk.so; fi
GP_LIB=$L timeout 600 python bench.py --no-pipeline > gpurun_out/bench_$n.json 2> gpurun_out/bench_$n.err; echo $n=$?
done
