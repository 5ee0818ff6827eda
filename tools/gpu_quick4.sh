# Quick: build, parity + full-size tests, bench of $CONFIGS.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/q4_tests.log 2>&1; tail -2 gpurun_out/q4_tests.log
for c in ${CONFIGS:-2 3 4 6}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python tools/bench_table.py gpurun_out/bench_c$c.json
done
