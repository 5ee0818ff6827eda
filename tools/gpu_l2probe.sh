# ncu of the gather-only probe on configs $CONFIGS (L2 hit rate of the A_hat^T gathers)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
M=$(python -c "import sys; sys.path.insert(0,'tools'); import l2_probe; print(','.join(l2_probe.METRICS))")
for c in ${CONFIGS:-2 3 4 5}; do
  python tools/l2_probe.py --config $c > gpurun_out/probe_plain_c$c.log 2>&1 &&
  ncu --metrics $M --clock-control none -k regex:k_gather_probe --csv python tools/l2_probe.py --config $c > gpurun_out/probe_ncu_c$c.csv 2>&1
  python tools/l2_probe.py --config $c --summarize gpurun_out/probe_ncu_c$c.csv --out gpurun_out
done
