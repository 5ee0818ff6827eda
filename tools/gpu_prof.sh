# Profiling pass: launch lists (all configs) + ncu --set full of the top kernels.
# Each ncu command runs only after the same command exited 0 without ncu.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 --clock-ms 0"
for c in 2 3 4 5; do
  $B --config $c > gpurun_out/plain_c$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv \
      $B --config $c > gpurun_out/ncu_launch_c$c.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:"k_num_merge|k_bucket_scatter|k_bucket_sort|k_analyze_sym|k_col_hist" \
    -s 5 -c 5 -o gpurun_out/full_c2 $B --config 2 > gpurun_out/ncu_full_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_num_warp|k_sym_warp|k_count_kept|k_compact_move|k_bucket_scatter|k_bucket_sort" \
    -s 6 -c 6 -o gpurun_out/full_c5 $B --config 5 > gpurun_out/ncu_full_c5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_num_huge|k_sym_huge|k_num_warp|k_analyze_sym" \
    -s 8 -c 8 -o gpurun_out/full_c4 $B --config 4 > gpurun_out/ncu_full_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_num_merge|k_analyze_sym|k_bucket_scatter|k_bucket_sort" \
    -s 4 -c 4 -o gpurun_out/full_c3 $B --config 3 > gpurun_out/ncu_full_c3.log 2>&1
ls -la gpurun_out
