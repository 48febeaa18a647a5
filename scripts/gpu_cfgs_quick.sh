# quick A/B: configs 1 and 2 (strict), device value + eval ms
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in ${CFGS:-1 2}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/q_c$c.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/q_c$c.json').read().strip().splitlines()[-1]);print('config $c', round(d['value'],1), 'eval_ms', round(d['roofline']['eval_ms_per_launch'],3), 'frac', round(d['roofline']['frac'],3))"
done
