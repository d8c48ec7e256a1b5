cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_build -s 1 -c 1 -o gpurun_out/prof_build_$1 python scripts/prof_run.py 10 > /dev/null 2>&1
ls gpurun_out
