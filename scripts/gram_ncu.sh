# ncu --set full capture of the fused cov/corr kernel (source-level), tuning aid
mkdir -p gpurun_out
make -j8 > /dev/null 2>&1
TAG=${1:-g2}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gram_fused -s 2 -c 1 -o gpurun_out/${TAG}_gram -f python scripts/gram_timing.py > gpurun_out/${TAG}_ncu.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/${TAG}_ncu.log
ls -la gpurun_out/${TAG}_gram.ncu-rep
