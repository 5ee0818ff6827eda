# ncu --set full of kernels matching $KREGEX on bench config $CFG (after a plain run).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 --clock-ms 0 --config ${CFG:-2}"
$B > gpurun_out/plain_ncu.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:"${KREGEX}" -s ${SKIP:-2} -c ${COUNT:-1} \
    -o gpurun_out/${OUT:-prof} $B > gpurun_out/ncu_${OUT:-prof}.log 2>&1
tail -3 gpurun_out/ncu_${OUT:-prof}.log
