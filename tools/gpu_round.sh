# Round evidence: parity tests, every config's bench line, the default bench
# (with the CPU oracle beside it), launch lists and ncu --set full captures.
set -x
mkdir -p gpurun_out
CONFIGS="${BENCH_CONFIGS:-2 3 4 5 1 6 7}" bash tools/gpu_test.sh
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
CONFIGS="2 3 4 5 6 7" bash tools/gpu_launches.sh
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 --clock-ms 0"
ncu --set full --import-source on --clock-control none -k regex:"k_num_pair|k_bucket_scatter|k_bucket_sort<|k_analyze_sym" -s 4 -c 4 -o gpurun_out/full_c2 $B --config 2 > gpurun_out/ncu_full_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_num_mid" -s 0 -c 1 -o gpurun_out/full_c5 $B --config 5 > gpurun_out/ncu_full_c5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_num_huge|k_num_mid|k_num_pair" -s 0 -c 4 -o gpurun_out/full_c4 $B --config 4 > gpurun_out/ncu_full_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_num_pair|k_analyze_sym|k_sym_transpose|k_row_norms" -s 4 -c 4 -o gpurun_out/full_c3 $B --config 3 > gpurun_out/ncu_full_c3.log 2>&1
ls gpurun_out
