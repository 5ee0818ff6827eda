# Mixed path: f_i threshold between the row-window kernel (temp mode) and the CTA-per-row kernel (RIG_CTA_MINF).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for c in 4 6; do for v in 256 192 160 128 256; do
  RIG_CTA_MINF=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "cfg $c minf=$v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'numeric', round(p.get('numeric',0),3))")"
done; done
