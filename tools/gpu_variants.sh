# Bench variants of librig (variants/NAME.so, built by tools/build_variant.sh) on $CONFIGS, $REPS rounds.
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for rep in $(seq ${REPS:-2}); do
for v in ${VARIANTS:-base}; do
  for c in ${CONFIGS:-2 3}; do
    if [ $v = base ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$PWD/variants/$v.so; fi
    python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
    echo "$v $(python tools/bench_table.py gpurun_out/v.json | cut -c1-70) $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);print(d['pass_ms']['numeric_kernel'], d['clocks']['sm_mhz'])")"
  done
done
done
