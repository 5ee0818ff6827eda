# Shared-memory CTA launch: longest-first threshold (RIG_CTA_BIGF0; 0 = one round) on configs 4, 6.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests -x -q -m gpu -k "long or cta or mixed or random_mixed" 2>&1 | tail -1
for c in 4 6; do for v in 0 512 768 1024 0; do
  RIG_CTA_BIGF0=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  echo "cfg $c bigf0=$v $(python -c "import json;d=json.loads(open('gpurun_out/v.json').read().splitlines()[-1]);p=d['pass_ms'];print(round(d['ms_per_step'],3), 'numeric', round(p.get('numeric',0),3))")"
done; done
