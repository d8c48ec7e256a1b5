cd $GRAFT_REPO_ROOT
b() { python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-c5-base 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['stage_ms_per_step']['force'], d['clocks'])"; }
b fresh1; b fresh2
timeout 300 python -m pytest tests/test_gpu_scale.py -q 2>&1 | tail -1
b after_tests
nvidia-smi --query-gpu=temperature.gpu,clocks.sm,power.draw --format=csv
