cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for s in "100 10" "200 20"; do set -- $s
 (cd abtest/v4 && python bench.py --steps $1 --warmup $2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.readline());print('v4',$1,d['value'],d['stage_ms_per_step'],d['roofline']['mean_row'])")
 python bench.py --steps $1 --warmup $2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.readline());print('head',$1,d['value'],d['stage_ms_per_step'],d['roofline']['mean_row'])"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_force -s 6 -c 1 -o gpurun_out/force_src python bench.py --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>gpurun_out/ncu.err
ls -la gpurun_out
