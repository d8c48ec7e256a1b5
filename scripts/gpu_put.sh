# ghost-update put A/B: domain + mock-NCCL suites, then the 1-GPU brick bench with puts and with pack/copy/unpack
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_domain.py tests/test_gpu_nccl_mock.py -q -x 2>&1 | tail -3
for p in 1 0; do
  echo "DPDB_PUT=$p"
  DPDB_PUT=$p timeout 600 python scripts/bench_bricks_1gpu.py 50 2>&1 | tail -8 | tee gpurun_out/bricks_put$p.jsonl
done
