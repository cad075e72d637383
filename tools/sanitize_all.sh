# compute-sanitizer over tools/sanitize_run.py (every kernel family and
# schedule); logs under gpurun_out/san/, stamped with the commit and the
# device-code hash.  Run on a GPU box:  bash tools/sanitize_all.sh
mkdir -p gpurun_out/san
{ git rev-parse HEAD 2>/dev/null || cat .git_head 2>/dev/null; python -c "import sys; sys.argv=['x']; sys.path.insert(0, '.'); import bench; print(bench.lib_sha256())"; } > gpurun_out/san/STAMP.txt
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/san/$t.txt 2>&1
  echo "$t rc=$?"; tail -2 gpurun_out/san/$t.txt
done
GPP_COLUMN_UPLOAD=1 timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/san/memcheck_column_upload.txt 2>&1
echo "memcheck (column upload) rc=$?"; tail -2 gpurun_out/san/memcheck_column_upload.txt
