# A/B one build under env settings: bash scripts/gpu_envab.sh "A=1" "A=0" ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do
  for e in "$@"; do
    env $e python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/envab.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/envab.json'));print('$e', d['value'], d['stage_ms_per_step'])"
  done
done
