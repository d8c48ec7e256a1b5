cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_force -s 3 -c 1 -o gpurun_out/prof_force2 python scripts/prof_run.py 10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_build -s 1 -c 1 -o gpurun_out/prof_build2 python scripts/prof_run.py 10 > /dev/null 2>&1
ls -la gpurun_out
