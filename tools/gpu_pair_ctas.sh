# k_num_pair resident CTAs per SM (RIG_PAIR_CTAS) on the merge-path configs.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for spec in "3:4" "3:5" "3:6" "3:0" "2:5" "2:6" "2:7" "2:0" "4:4" "4:5"; do
  c=${spec%%:*}; v=${spec#*:}
  RIG_PAIR_CTAS=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>/dev/null
  echo "cfg $c ctas=$v $(python -c "import json;d=json.loads(open('gpurun_out/b.json').read().splitlines()[-1]);print(round(d['ms_per_step'],3), round(d['pass_ms'].get('numeric_kernel',0),4), round(d['pass_ms']['numeric'],3))")"
done
