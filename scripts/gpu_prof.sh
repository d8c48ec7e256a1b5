cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_run.py 10 > gpurun_out/prof_run.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_force -s 3 -c 1 -o gpurun_out/prof_force python scripts/prof_run.py 10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_build -s 1 -c 1 -o gpurun_out/prof_build python scripts/prof_run.py 10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_radix|k_scan|k_permute" -s 0 -c 6 -o gpurun_out/prof_sort python scripts/prof_run.py 10 > /dev/null 2>&1
ls -la gpurun_out
