# A/B environment settings on one box: bash scripts/gpu_envab.sh "NAME:ENV=V ENV2=V" ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  for r in 1 2; do
    env $envs python bench.py --steps ${STEPS:-100} --warmup 10 --no-cpu-baseline > gpurun_out/envab_${name}_$r.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/envab_${name}_$r.json'));print('$name', d['value'], d['stage_ms_per_step'])"
  done
done
