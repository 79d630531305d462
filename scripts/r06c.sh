set -x
mkdir -p gpurun_out
make -j8 > /dev/null 2>&1
for k in conv2d conv3d fdtd_2d; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${k%_2d}" -s 2 -c 1 -o gpurun_out/r06_${k} -f python scripts/stencil_one.py $k 3 > gpurun_out/r06_${k}_ncu.log 2>&1
  tail -2 gpurun_out/r06_${k}_ncu.log
done
ls -la gpurun_out | grep r06_
