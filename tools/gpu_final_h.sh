# Launch lists of every config and the ncu --set full capture of config 5's transpose kernels (final code).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
CONFIGS="2 3 4 5 6 7" bash tools/gpu_launches.sh > /dev/null 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 --clock-ms 0"
ncu --set full --import-source on --clock-control none -k regex:"k_bucket_scatter|k_bucket_sort|k_col_hist" -s 3 -c 4 -o gpurun_out/full_c5t_h $B --config 5 > gpurun_out/ncu_full_c5t_h.log 2>&1
ls gpurun_out | grep -c launches
