# paper-size sweep + compute-sanitizer (memcheck / racecheck / synccheck) over smoke()
timeout 900 python scripts/paper_sizes.py gpurun_out/paper_sizes.json 2>&1 | tail -12
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
     python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done
