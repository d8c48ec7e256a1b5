# A/B library builds on one box: bash scripts/gpu_ab.sh NAME... (abtest/NAME.so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_1311_0402_b200/libdpdb.so /tmp/libdpdb_keep.so
for v in "$@"; do
  cp abtest/$v.so paper_1311_0402_b200/libdpdb.so
  for r in 1 2; do
    python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/ab_${v}_$r.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$r.json'));print('$v', d['value'], d['stage_ms_per_step'])"
  done
done
cp /tmp/libdpdb_keep.so paper_1311_0402_b200/libdpdb.so
