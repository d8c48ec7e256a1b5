# A/B library builds on selected configs: CONFIGS=C4 bash scripts/gpu_ab_cfg2.sh NAME...
cd $GRAFT_REPO_ROOT
cp paper_1311_0402_b200/libdpdb.so /tmp/libdpdb_keep.so
for v in "$@"; do
  cp abtest/$v.so paper_1311_0402_b200/libdpdb.so
  python scripts/bench_configs.py 100 2>/dev/null | sed "s/^/$v /" | cut -c1-260
done
cp /tmp/libdpdb_keep.so paper_1311_0402_b200/libdpdb.so
