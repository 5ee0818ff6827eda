# Performance experiments: bench config $CFG under several RIG_DEBUG_MASK values (results not checked).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for m in ${MASKS:-0}; do
  RIG_DEBUG_MASK=$m timeout 300 python bench.py --config ${CFG:-5} --steps 5 --warmup 3 --no-cpu-baseline --soak-seconds 0.5 > gpurun_out/dbg_$m.json 2> gpurun_out/dbg_$m.err
done
