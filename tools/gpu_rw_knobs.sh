# Row-window knobs on config 5: no L2 prefetch of the next row's columns
# (RIG_DEBUG_MASK=4), unit-table and far-list capacities.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh tcap32 "-DRIG_RW_TCAP=32" > /dev/null 2>&1 &
bash tools/build_variant.sh fcap160 "-DRIG_RW_FCAP=160" > /dev/null 2>&1 &
bash tools/build_variant.sh fcap224 "-DRIG_RW_FCAP=224" > /dev/null 2>&1 &
wait
for rep in 1 2; do for v in base nopf tcap32 fcap160 fcap224; do
  unset RIG_LIB_VARIANT RIG_DEBUG_MASK
  case $v in base) ;; nopf) export RIG_DEBUG_MASK=4;; *) export RIG_LIB_VARIANT=$PWD/variants/$v.so;; esac
  timeout 300 python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'kernel', round(p.get('numeric_kernel',0),3))")"
done; done
