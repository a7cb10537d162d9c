# parity tests + timeline + graph timing of the default build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/gpu_tests.log
python scripts/warp_timeline.py > gpurun_out/tl.log 2>&1
GT_SHAPES=${GT_SHAPES:-56x56,28x28,2048x7,small,bf16} timeout 300 python scripts/graph_timing.py ${GT_RATIOS:-10,100,1000} > gpurun_out/gt_default.log 2>&1; echo gt=$?
