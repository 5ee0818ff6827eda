# ncu --set full (source-level) of config 5's row-window kernel and its transpose
# scatter/sort, for per-line instruction and stall attribution (tools/ncu_lines2.py).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 --clock-ms 0"
$B --config 5 > gpurun_out/plain_c5.log 2>&1 || { tail gpurun_out/plain_c5.log; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:"k_row_win|k_bucket_scatter|k_bucket_sort" -s 3 -c 3 \
    -o gpurun_out/src_c5 $B --config 5 > gpurun_out/ncu_src_c5.log 2>&1
tail -3 gpurun_out/ncu_src_c5.log
