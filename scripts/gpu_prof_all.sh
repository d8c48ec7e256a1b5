# ncu evidence for the current build: launch list + full captures of the hot kernels
# usage: bash scripts/gpu_prof_all.sh TAG   (then: python scripts/ncu_summary.py TAG)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/prof_run.py 20 > /dev/null 2>&1
# 4th pair-force launch = step 3: the fused Verlet-epilogue variant (streams)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_force -s 3 -c 1 -o gpurun_out/full_force_$TAG python scripts/prof_run.py 10 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_build -s 1 -c 1 -o gpurun_out/full_build_$TAG python scripts/prof_run.py 10 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_onesweep|k_permute" -s 0 -c 5 -o gpurun_out/full_sort_$TAG python scripts/prof_run.py 10 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_integrate -s 0 -c 1 -o gpurun_out/full_integrate_$TAG python scripts/prof_run.py 10 > /dev/null 2>&1
ls gpurun_out | grep $TAG
