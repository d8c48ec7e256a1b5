# GPU validation cycle: the -m gpu suite (summary) + one bench line (stages)
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -${TAILN:-6}
python bench.py --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('BENCH', d['value'], 'ms/step', d['ms_per_step'], d['stage_ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'clk', d.get('clocks'))"
