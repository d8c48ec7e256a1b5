# GPU check: parity suite + bench (no CPU baseline) -- usage: bash scripts/gpu_check.sh TAG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-x}
python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/pytest_$T.log
cat gpurun_out/pytest_$T.log
python bench.py --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
python -c "import json;d=json.load(open('gpurun_out/bench_$T.json'));print(d['value'],d['stage_ms_per_step'],d['roofline']['frac'],d['e2e']['value'])" || tail -20 gpurun_out/bench_$T.err
