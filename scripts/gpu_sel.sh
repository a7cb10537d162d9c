cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in x10 x11 x12 x1 x2; do
GP_LIB=paper_2410_12707_b200/_lib/variants/$n/libadatopk.so GT_COMPRESS_ONLY=1 GT_SHAPES=2048x7,56x56 timeout 300 python scripts/graph_timing.py 1000 > gpurun_out/gt_$n.log 2>&1; echo $n=$?
done
