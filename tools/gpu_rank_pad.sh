# Small-bucket transpose sort: padded, 16-byte aligned key copies so the rank
# loop compares four keys per shared load (RIG_RANK_PAD=1) vs the scalar loop.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh rankpad "-DRIG_RANK_PAD=1" > gpurun_out/rankpad_build.log 2>&1 || { tail gpurun_out/rankpad_build.log; exit 1; }
for rep in 1 2; do for c in 5 7 6; do for v in base rankpad; do
  unset RIG_LIB_VARIANT
  case $v in base) ;; *) export RIG_LIB_VARIANT=$PWD/variants/$v.so;; esac
  timeout 300 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "c$c $v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'scatter+sort', round(p.get('scale_scatter',0),3))")"
done; done; done
export RIG_LIB_VARIANT=$PWD/variants/rankpad.so
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/rankpad_tests.log 2>&1; tail -2 gpurun_out/rankpad_tests.log
