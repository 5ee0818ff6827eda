# Row-window kernel experiments: parity tests of the row-window path, then
# config-5 bench of librig variants ($VARS: "name:defines;name:defines").
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-row_window or small_configs}" > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
names="base"
IFS=';' read -ra VV <<< "$VARS"
for v in "${VV[@]}"; do
  n=${v%%:*}; d=${v#*:}
  bash tools/build_variant.sh $n "$d" > /dev/null 2>&1 &
  names="$names $n"
done
wait
VARIANTS="$names" CONFIGS="${CONFIGS:-5}" REPS=${REPS:-2} bash tools/gpu_variants.sh
