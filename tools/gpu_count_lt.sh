# Rank loops with compare + predicated increment (count_lt): every config, then the gpu tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || { tail gpurun_out/smoke.log; exit 1; }
tail -1 gpurun_out/smoke.log
rm -f gpurun_out/rc_bench_all_configs.jsonl
for c in 1 2 3 4 5 6 7; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bc$c.json 2> gpurun_out/bc$c.err
  tail -1 gpurun_out/bc$c.json >> gpurun_out/rc_bench_all_configs.jsonl
  python -c "import json;d=json.loads(open('gpurun_out/bc$c.json').read().splitlines()[-1]);p=d['pass_ms'];print($c, round(d['ms_per_step'],4), 'scatter+sort', round(p.get('scale_scatter',0),4))"
done
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
CONFIGS="5" bash tools/gpu_launches.sh > /dev/null 2>&1
