# Quick: build, parity tests, bench of configs 1 2 5 with the launch list of config 2.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/q3_tests.log 2>&1; tail -1 gpurun_out/q3_tests.log
for c in 1 2 3 5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python tools/bench_table.py gpurun_out/bench_c$c.json
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tile_sum|k_tile_scan|k_col_hist" --csv python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 --clock-ms 0 2>/dev/null | grep -o '"k_[a-z_]*[^"]*","[^"]*","[^"]*","[^"]*"' | tail -6
