# Row-window staged copy: rounds per iteration (RIG_RW_COPYU) and ring depth on config 5.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh cu2 "-DRIG_RW_COPYU=2" > /dev/null 2>&1 &
bash tools/build_variant.sh cu4 "-DRIG_RW_COPYU=4" > /dev/null 2>&1 &
bash tools/build_variant.sh d2 "-DRIG_RW_DEPTH=2" > /dev/null 2>&1 &
wait
for rep in 1 2; do for v in base cu2 cu4 d2; do
  if [ $v = base ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'kernel', round(p.get('numeric_kernel',0),3))")"
done; done
