# library -D knob variants (VS="a b", built by build_variant.py): parity tests per variant, then N=1 bench alternating default/variants (development aid)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
VS=${VS:-"t32b2 t8b4 t16b3 t8b3"}
for V in $VS; do
  echo "== parity $V"
  GP_LIB=paper_2410_12707_b200/_lib/variants/$V/libadatopk.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
done
for r in 1 2; do
for V in default $VS; do
  L=$([ $V = default ] && echo "" || echo paper_2410_12707_b200/_lib/variants/$V/libadatopk.so)
  GP_LIB=$L timeout 300 python bench.py --no-pipeline > gpurun_out/knob_${V}_$r.json 2>/dev/null
  python -c "import json;j=json.loads(open('gpurun_out/knob_${V}_$r.json').read().splitlines()[-1]);print('$V $r', j['value'], j['ms_per_step'], j['roofline']['achieved'], j['roofline']['decompress_achieved'], j['c1_gpt2_small']['pair_us'])"
done
done
