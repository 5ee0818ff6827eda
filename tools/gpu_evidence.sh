# Round evidence (final code): every gpu test, every config's bench line, the default
# bench (with the CPU oracle beside it), the reference arm, launch lists and
# ncu --set full captures of the dominant kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
rm -f gpurun_out/rc_bench_all_configs.jsonl
for c in 1 2 3 4 5 6 7; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bc$c.json 2> gpurun_out/bc$c.err
  tail -1 gpurun_out/bc$c.json >> gpurun_out/rc_bench_all_configs.jsonl
done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
# the N > 1 bench path (row shards + allreduce) with 2 ranks sharing the one GPU (gloo): a path check, not a number
BENCH_SHARE_GPU=1 BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2ranks_shared.json 2> gpurun_out/bench_2ranks_shared.err
CONFIGS="2 3 4 5 6 7" bash tools/gpu_launches.sh > /dev/null 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 --clock-ms 0"
ncu --set full --import-source on --clock-control none -k regex:"k_row_win" -s 1 -c 1 -o gpurun_out/full_c5 $B --config 5 > gpurun_out/ncu_full_c5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_num_pair|k_bucket_scatter|k_bucket_sort|k_analyze_sym" -s 4 -c 4 -o gpurun_out/full_c2 $B --config 2 > gpurun_out/ncu_full_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_num_pair|k_analyze_sym|k_sym_transpose|k_row_norms" -s 4 -c 4 -o gpurun_out/full_c3 $B --config 3 > gpurun_out/ncu_full_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_row_win|k_row_cta|k_num_huge|k_num_mid|k_num_pair|k_copy_rows" -s 0 -c 8 -o gpurun_out/full_c4 $B --config 4 > gpurun_out/ncu_full_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_bucket_scatter|k_bucket_sort|k_col_hist" -s 3 -c 4 -o gpurun_out/full_c5t $B --config 5 > gpurun_out/ncu_full_c5t.log 2>&1
ls gpurun_out | head -80
