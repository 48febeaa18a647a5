# round-end evidence refresh (one GPU): launch list + ncu captures (configs 2, 1, 3, 4), bench lines -> gpurun_out/; then scripts/update_profiles.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=r02 bash scripts/gpu_profile_round.sh
for c in 1 3 4; do CFG=$c TAG=c${c}f bash scripts/gpu_ncu_env.sh; done
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
for c in 1 3 4; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo c$c rc=$?; done
python bench.py --precision fast --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fast.json 2> gpurun_out/bench_fast.err; echo fast rc=$?
