# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_driver.py (small inputs)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for t in ${TOOLS:-memcheck racecheck synccheck}; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_driver.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; tail -4 gpurun_out/sanitize_$t.log
done
