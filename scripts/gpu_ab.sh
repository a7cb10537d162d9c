# A/B: default lib + variants under _lib/variants/*, graph timing each
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
timeout 300 python scripts/graph_timing.py > gpurun_out/gt_default.log 2>&1; echo default=$?
for v in paper_2410_12707_b200/_lib/variants/*/; do n=$(basename $v)
GP_LIB=$v/libadatopk.so timeout 300 python scripts/graph_timing.py > gpurun_out/gt_$n.log 2>&1; echo $n=$?
done
