# targeted ncu metrics of the fused force kernel for several library builds: bash scripts/gpu_ncu_ab.sh NAME...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_1311_0402_b200/libdpdb.so /tmp/libdpdb_keep.so
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct
for v in "$@"; do
  cp abtest/$v.so paper_1311_0402_b200/libdpdb.so
  timeout 300 ncu --metrics $M --clock-control none -k regex:k_force_walk -s 3 -c 1 --csv python scripts/prof_run.py 5 2>/dev/null | grep "^\"" > gpurun_out/ncuab_$v.csv
  echo "== $v"; python -c "
import csv,sys
r=list(csv.reader(open('gpurun_out/ncuab_$v.csv')))
h=r[0]; i=h.index('Metric Name'); j=h.index('Metric Value')
for x in r[1:]: print('  ',x[i],x[j])"
done
cp /tmp/libdpdb_keep.so paper_1311_0402_b200/libdpdb.so
