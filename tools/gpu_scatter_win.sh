# Transpose scatter: windowed bucket reservation (RIG_SCATTER_WIN, V chunks per
# sub-tile, RIG_SCATTER_MINB register cap) vs the per-chunk-group atomics (WIN=0).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh w0 "-DRIG_SCATTER_WIN=0" > /dev/null 2>&1 &
bash tools/build_variant.sh v4m4 "-DRIG_SCATTER_V=4 -DRIG_SCATTER_MINB=4" > /dev/null 2>&1 &
bash tools/build_variant.sh v8m3 "-DRIG_SCATTER_V=8 -DRIG_SCATTER_MINB=3" > /dev/null 2>&1 &
bash tools/build_variant.sh v8 "-DRIG_SCATTER_V=8" > /dev/null 2>&1 &
bash tools/build_variant.sh v2 "-DRIG_SCATTER_V=2" > /dev/null 2>&1 &
wait
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/sw_tests.log 2>&1; tail -1 gpurun_out/sw_tests.log
for c in 5 2 4; do for v in base w0 v4m4 v8m3 v8 v2; do
  if [ $v = base ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "cfg $c $v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'scatter', round(p.get('scale_scatter',0),3), 'colptr', round(p.get('colptr',0),3))")"
done; done
