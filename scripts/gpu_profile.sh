# ncu evidence for profiles/: launch list of the bench command + full captures of the hot kernels
TAG=${1:-r03}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-next --graphs 0 > gpurun_out/${TAG}_ncu_bench.log 2>&1
cap() {  # name kernel-regex skip bench-kernels
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/${TAG}_$1 -f \
     python bench.py --kernels $4 --steps 1 --warmup 3 --no-e2e --no-cpu --graphs 0 > /dev/null 2>&1
}
cap syr2k umma3x 3 syr2k
cap 2mm umma3x 6 2mm
cap atax atax 3 atax
cap bicg mvmt 3 bicg
cap gesummv gesummv_tile 3 gesummv
cap cov_gram umma3x 3 covariance
cap cov_prep band_prep 3 covariance
cap cov_combine gram_combine 3 covariance
ls gpurun_out | grep $TAG
