# Small-bucket transpose sort on config 5 (and 7): rank vs per-lane insertion sorts.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash tools/build_variant.sh srank0 "-DRIG_SMALL_RANK=0" > /dev/null 2>&1
for rep in 1 2; do for c in 5 7; do for v in base srank0; do
  unset RIG_LIB_VARIANT
  case $v in base) ;; *) export RIG_LIB_VARIANT=$PWD/variants/$v.so;; esac
  timeout 300 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "c$c $v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'scatter+sort', round(p.get('scale_scatter',0),3))")"
done; done; done
