mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "small_configs or row_window or mid_rows or build_cut or shards" > gpurun_out/t1.log 2>&1; tail -5 gpurun_out/t1.log
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b5.json 2> gpurun_out/b5.err; tail -c 1500 gpurun_out/b5.json; tail -3 gpurun_out/b5.err
