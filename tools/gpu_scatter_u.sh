# Transpose scatter: chunks per group (RIG_SCATTER_U) variants on configs 5, 2, 4.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh u4 "-DRIG_SCATTER_U=4" > /dev/null 2>&1 &
bash tools/build_variant.sh u3 "-DRIG_SCATTER_U=3" > /dev/null 2>&1 &
bash tools/build_variant.sh u6 "-DRIG_SCATTER_U=6" > /dev/null 2>&1 &
wait
for c in 5 2 4; do for v in base u3 u4 u6; do
  if [ $v = base ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "cfg $c $v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'scatter', round(p.get('scale_scatter',0),3), 'colptr', round(p.get('colptr',0),3))")"
done; done
