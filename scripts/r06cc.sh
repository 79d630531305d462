make -j8 > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  PB_C3_RPW=2 timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_next.py > gpurun_out/r06_sanitizer_next_$tool.log 2>&1; echo $tool rc=$?
  tail -2 gpurun_out/r06_sanitizer_next_$tool.log
done
timeout 900 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r06_sanitizer_smoke_memcheck.log 2>&1; echo smoke-memcheck rc=$?
tail -2 gpurun_out/r06_sanitizer_smoke_memcheck.log
