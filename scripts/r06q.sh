make -j8 > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_next.py > gpurun_out/r06_sanitizer_next_$tool.log 2>&1; echo $tool rc=$?
  tail -4 gpurun_out/r06_sanitizer_next_$tool.log
done
