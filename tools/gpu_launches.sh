# Launch list (ncu gpu__time_duration only) of bench configs $CONFIGS, after a plain run each.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in ${CONFIGS:-2}; do
  B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 --clock-ms 0 --config $c"
  $B > gpurun_out/plain_c$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv $B > gpurun_out/ncu_launch_c$c.log 2>&1
done
