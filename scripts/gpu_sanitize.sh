# compute-sanitizer memcheck / racecheck / synccheck / initcheck over scripts/sanitize_run.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/sanitize_run.py > gpurun_out/san_plain.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
      python scripts/sanitize_run.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -c '^ok' gpurun_out/san_$tool.txt) stages; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_$tool.txt | tail -2 | tr '\n' ' ')"
done
