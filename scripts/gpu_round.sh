cd $GRAFT_REPO_ROOT
bash scripts/gpu_check.sh v5
python bench.py > gpurun_out/bench_full_v5.json 2> gpurun_out/bench_full_v5.err
bash scripts/gpu_prof_all.sh v5
