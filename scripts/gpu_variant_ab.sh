# graph_timing (GPT-2 + ResNet shapes) and the N=1 bench, default build vs one variant, alternating (development aid)
#   V=defer bash scripts/gpu_variant_ab.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
V=${V:-defer}
for r in 1 2; do
for L in "" paper_2410_12707_b200/_lib/variants/$V/libadatopk.so; do
tag=$([ -z "$L" ] && echo default || echo $V)
echo "== $tag $r"
GP_LIB=$L timeout 300 python scripts/graph_timing.py ${RATIOS:-100} 2>&1 | grep -v "^ *warm\|phase" | cut -c1-200
GP_LIB=$L timeout 300 python bench.py --no-pipeline > gpurun_out/vab_${tag}_$r.json 2>/dev/null; python -c "import json;j=json.loads(open('gpurun_out/vab_${tag}_$r.json').read().splitlines()[-1]);print('bench', j['value'], j['ms_per_step'], j['c1_gpt2_small']['pair_us'], j['c1_gpt2_small']['batch8_8streams']['frac_of_peak'])"
done
done
