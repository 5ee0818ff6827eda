# quick: selected parity tests + config-5 bench (no cpu baseline)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "${TESTK:-small_configs or row_window or mid_rows}" > gpurun_out/t1.log 2>&1; tail -3 gpurun_out/t1.log
for c in ${CONFIGS:-5}; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b$c.json 2> gpurun_out/b$c.err
python - <<PY
import json
d=json.loads(open("gpurun_out/b$c.json").read().strip().splitlines()[-1])
print($c, "ms/step", round(d["ms_per_step"],3), "numeric", round(d["numeric_ms"],3), "kernel", round(d["numeric_kernel_ms"],3), "frac", round(d["roofline"]["frac"],3), {k:round(v,3) for k,v in d["pass_ms"].items()})
PY
done
