# A/B the force kernel of two library builds on the same box
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  cp abtest/$v.so paper_1311_0402_b200/libdpdb.so
  for r in 1 2; do
    python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/ab_$v_$r.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_$v_$r.json'));print('$v', d['value'], d['stage_ms_per_step'])"
  done
done
