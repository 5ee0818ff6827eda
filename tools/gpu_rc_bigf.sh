# RANGE launch: threshold of the longest-first round (RIG_RC_BIGF) on configs 4, 6.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh b4k "-DRIG_RC_BIGF=4096" > /dev/null 2>&1 &
bash tools/build_variant.sh b16k "-DRIG_RC_BIGF=16384" > /dev/null 2>&1 &
bash tools/build_variant.sh b2k "-DRIG_RC_BIGF=2048" > /dev/null 2>&1 &
wait
for c in 4 6; do for v in base b2k b4k b16k; do
  if [ $v = base ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "cfg $c $v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'numeric', round(p.get('numeric',0),3))")"
done; done
