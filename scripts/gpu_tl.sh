cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in ${TL_VARIANTS:-default st1 st2 st3 noproc}; do
if [ $n = default ]; then L=""; else L=paper_2410_12707_b200/_lib/variants/$n/libadatopk.so; fi
echo "=== $n"; GP_LIB=$L python scripts/warp_timeline.py ${TL_ARGS:-}
done > gpurun_out/tl.log 2>&1
