# round evidence: parity suite, full bench (with the CPU baseline), reference arm, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-round}
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_$T.log
cat gpurun_out/pytest_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
bash scripts/gpu_prof_all.sh $T
