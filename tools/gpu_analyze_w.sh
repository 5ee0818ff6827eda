# Analysis kernel: merge width per warp (RIG_ANALYZE_WARP_WIDTH=1, default) vs per
# lane (0), and register caps (RIG_ANALYZE_MINB), on the configs that analyse.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh aw0 "-DRIG_ANALYZE_WARP_WIDTH=0" > /dev/null 2>&1 &
bash tools/build_variant.sh am3 "-DRIG_ANALYZE_MINB=3" > /dev/null 2>&1 &
bash tools/build_variant.sh aw0m3 "-DRIG_ANALYZE_WARP_WIDTH=0 -DRIG_ANALYZE_MINB=3" > /dev/null 2>&1 &
wait
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/aw_tests.log 2>&1; tail -1 gpurun_out/aw_tests.log
for c in 3 2 4; do for v in base aw0 am3 aw0m3 base aw0; do
  if [ $v = base ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "cfg $c $v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'analyze', round(p.get('analyze',0),3), 'numeric', round(p.get('numeric',0),3))")"
done; done
