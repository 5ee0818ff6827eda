# Merge kernel register budget variants (RIG_PAIR_MINB) on configs 2, 3.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh m8 "-DRIG_PAIR_MINB=8" > /dev/null 2>&1 &
bash tools/build_variant.sh m7 "-DRIG_PAIR_MINB=7" > /dev/null 2>&1 &
bash tools/build_variant.sh t256 "-DRIG_PAIR_THREADS=256" > /dev/null 2>&1 &
wait
for c in 2 3; do for v in base m7 m8 t256; do
  if [ $v = base ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "cfg $c $v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'kernel', round(p.get('numeric_kernel',0),4))")"
done; done
