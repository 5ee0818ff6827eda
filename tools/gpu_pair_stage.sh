# Merge kernel output stage size (RIG_PAIR_STAGE_F x 16 rows x mean products) on configs 2, 3.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh sf45 "-DRIG_PAIR_STAGE_F=0.45" > /dev/null 2>&1 &
bash tools/build_variant.sh sf52 "-DRIG_PAIR_STAGE_F=0.52" > /dev/null 2>&1 &
bash tools/build_variant.sh sf75 "-DRIG_PAIR_STAGE_F=0.75" > /dev/null 2>&1 &
wait
for c in 3 2; do for v in base sf45 sf52 sf75; do
  if [ $v = base ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "cfg $c $v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'kernel', round(p.get('numeric_kernel',0),4), 'numeric', round(p.get('numeric',0),4))")"
done; done
