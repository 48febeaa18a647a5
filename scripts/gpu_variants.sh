# A/B of prebuilt library variants: variants/libsqv_<name>.so -> bench (eval ms) + precision
# usage: bash scripts/gpu_variants.sh exp0 exp1 ...   (FIELD via env SQV_FIELD, default both 6 and 7)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
LIB=paper_2511_17361_b200/_build/libsqv.so
cp $LIB /tmp/libsqv_orig.so
for V in "$@"; do
  cp variants/libsqv_$V.so $LIB
  for F in ${FIELDS:-6 7}; do
    tag=${V}_f$F
    SQV_FIELD=$F timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_$tag.json 2>gpurun_out/var_$tag.err
    SQV_FIELD=$F timeout 600 python scripts/diag_precision.py > /dev/null 2>&1; cp gpurun_out/diag_precision.json gpurun_out/var_${tag}_prec.json
    python - $tag <<'PY'
import json,sys
tag=sys.argv[1]
d=json.loads(open(f"gpurun_out/var_{tag}.json").read().strip().splitlines()[-1])
p=json.load(open(f"gpurun_out/var_{tag}_prec.json"))
rows={k.replace("vo_",""):("%.1e"%v["rel_max"],v["n_over_1e-5"]) for k,v in p["vo_config1"].items()}
print(f"{tag}: value {d['value']:.1f} eval_ms {d['roofline']['eval_ms_per_launch']:.3f} frac {d['roofline']['frac']:.3f} | {rows}")
PY
  done
done
cp /tmp/libsqv_orig.so $LIB
