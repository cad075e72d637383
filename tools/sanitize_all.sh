mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/san/$t.txt 2>&1
  echo "$t rc=$?"; tail -2 gpurun_out/san/$t.txt
done
