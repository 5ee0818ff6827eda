# GPU parity + quick bench of every config (no ncu).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
for c in ${CONFIGS:-2 3 4 5 1}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
tail -3 gpurun_out/gputests.log
