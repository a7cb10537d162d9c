# A/B variants on the largest boundary only (fast), stamps included
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in default paper_2410_12707_b200/_lib/variants/*/; do
[ $v = default ] || [ -d "$v" ] || continue
n=$(basename $v)
if [ $v = default ]; then L=""; else L=$v/libadatopk.so; fi
GP_LIB=$L GT_SHAPES="${GT_SHAPES:-56x56}" timeout 300 python scripts/graph_timing.py ${GT_RATIOS:-10,100,1000} > gpurun_out/gt_$n.log 2>&1; echo $n=$?
done
