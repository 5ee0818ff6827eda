# Timing experiments on config $CFG: each line "label env..." runs bench.py once (results not checked).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
while read -r label envs; do
  [ -z "$label" ] && continue
  env $envs timeout 300 python bench.py --config ${CFG:-5} --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --soak-seconds 0.3 > gpurun_out/exp_$label.json 2> gpurun_out/exp_$label.err
  python - "$label" <<'PY'
import json, sys
lab = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/exp_{lab}.json").read().strip().splitlines()[-1])
    print(lab, "ms/step", round(d["ms_per_step"], 3), "numeric", round(d["numeric_ms"], 3),
          {k: round(v, 3) for k, v in d["pass_ms"].items()})
except Exception as e:
    print(lab, "FAILED", e, open(f"gpurun_out/exp_{lab}.err").read()[-800:])
PY
done < ${EXPS:-gpurun_out/exps.txt}
