cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 1 3 4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo c$c rc=$?
  python -c "import json;d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1]);print('config $c', round(d['value'],1), d['unit'], 'pairs/s %.3e'%d['pairs_per_s'], 'frac %.3f'%d['roofline']['frac'], 'e2e', round(d['e2e']['value'],1))"
done
timeout 900 python bench.py --precision fast --no-cpu-baseline > gpurun_out/bench_fast.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bench_fast.json').read().strip().splitlines()[-1]);print('config 2 fast', round(d['value'],1), 'frac %.3f'%d['roofline']['frac'], 'e2e', round(d['e2e']['value'],1))"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; echo torchrun rc=$?
tail -c 300 gpurun_out/bench_torchrun1.json
