# one iteration: parity suite, bench (no CPU baseline), ncu of the builder + force
# usage: bash scripts/gpu_iter.sh TAG [pytest-args]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-x}
shift
timeout 900 python -m pytest tests -m gpu -x -q ${@} 2>&1 | tail -15 > gpurun_out/pytest_$T.log
cat gpurun_out/pytest_$T.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
python -c "import json;d=json.load(open('gpurun_out/bench_$T.json'));print(d['value'],d['stage_ms_per_step'],d['roofline']['frac'],d['e2e']['value'])" || tail -20 gpurun_out/bench_$T.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_build -s 1 -c 1 -o gpurun_out/full_build_$T python scripts/prof_run.py 10 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_force -s 3 -c 1 -o gpurun_out/full_force_$T python scripts/prof_run.py 10 > /dev/null 2>&1
ls gpurun_out | tail -5
