# parity tests, then the bench alternating default / variants (2 rounds) to average out noise
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider ${GP_TESTS_K:+-k "$GP_TESTS_K"} > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
for r in 1 2; do
for v in default paper_2410_12707_b200/_lib/variants/*/; do
[ $v = default ] || [ -d "$v" ] || continue
n=$(basename $v)
if [ $v = default ]; then L=""; else L=$v/libadatopk.so; fi
GP_LIB=$L timeout 600 python bench.py --no-pipeline > gpurun_out/bench_${n}_$r.json 2> gpurun_out/bench_${n}_$r.err; echo $n$r=$? $(python -c "import json;j=json.loads(open('gpurun_out/bench_${n}_$r.json').read().splitlines()[-1]);print(j['value'],j['roofline']['frac'])")
done
done
