# ncu --set full with source counters of one k_force_walk launch (C3 bench)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-x}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:${2:-k_force_walk} -s ${3:-6} -c 1 -o gpurun_out/ncu_$T python bench.py --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_$T.err
ls -la gpurun_out/ncu_$T.ncu-rep
