# Merge width dispatch per lane (base) vs per warp (RIG_PAIR_WARP_DISPATCH=1).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh wd "-DRIG_PAIR_WARP_DISPATCH=1" > /dev/null 2>&1
RIG_LIB_VARIANT=$PWD/variants/wd.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "small_configs or random_mixed or build_cut" 2>&1 | tail -1
for c in 4 2 3 6; do for v in base wd; do
  if [ $v = base ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "cfg $c $v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'numeric', round(p.get('numeric',0),3), 'kernel', round(p.get('numeric_kernel',0),3))")"
done; done
