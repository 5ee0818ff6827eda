# Row-window far-sort knobs on config 5: 256 sort buckets (8 CTAs per SM by
# shared memory, 64-register budget) and the per-lane insertion-sort limit.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh nb256 "-DRIG_RW_NB=256 -DRIG_RW_MINB=8" > /dev/null 2>&1 &
bash tools/build_variant.sh minb8 "-DRIG_RW_MINB=8" > /dev/null 2>&1 &
bash tools/build_variant.sh sb16 "-DRIG_RW_SMALLB=16" > /dev/null 2>&1 &
bash tools/build_variant.sh sb4 "-DRIG_RW_SMALLB=4" > /dev/null 2>&1 &
wait
for rep in 1 2; do for v in base nb256 minb8 sb16 sb4; do
  unset RIG_LIB_VARIANT
  case $v in base) ;; *) export RIG_LIB_VARIANT=$PWD/variants/$v.so;; esac
  timeout 300 python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'kernel', round(p.get('numeric_kernel',0),3))")"
done; done
