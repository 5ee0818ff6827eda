python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "long or mixed or huge or parity_small or dist" > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
bash tools/build_variant.sh fw256 "-DRIG_RC_FW=256" > /dev/null 2>&1 &
bash tools/build_variant.sh fw192m3 "-DRIG_RC_FW=192 -DRIG_RC_MINB=3" > /dev/null 2>&1 &
bash tools/build_variant.sh fw128m4 "-DRIG_RC_FW=128 -DRIG_RC_MINB=4" > /dev/null 2>&1 &
wait
VARIANTS="base fw256 fw192m3 fw128m4" CONFIGS="4 6" REPS=1 bash tools/gpu_variants.sh
