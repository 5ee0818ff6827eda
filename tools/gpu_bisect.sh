# run test $TESTK against every variants/*.so and the default lib
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in default variants/*.so; do
  if [ "$v" = default ]; then unset RIG_LIB_VARIANT; else export RIG_LIB_VARIANT=$v; fi
  r=$(timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "$TESTK" 2>&1 | tail -1)
  echo "$v: $r"
done
