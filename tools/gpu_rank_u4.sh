# Bucket sort: the column-rank loop with four independent counts (RIG_RANK_U4=1)
# vs one count per loop trip (0), on the configs that rank (mean column > 12).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh r0 "-DRIG_RANK_U4=0" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/ru_tests.log 2>&1; tail -1 gpurun_out/ru_tests.log
for c in 5 7 6; do for v in base r0 base r0; do
  if [ $v = base ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "cfg $c $v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'scatter', round(p.get('scale_scatter',0),3), 'colptr', round(p.get('colptr',0),3))")"
done; done
