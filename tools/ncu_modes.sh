mkdir -p gpurun_out/h16j
for m in 7 32 0; do
  SST_DEBUG_MODE=$m timeout 300 ncu --set full --clock-control none -k regex:stencil_step -s 6 -c 1 -o gpurun_out/h16j/m$m python tools/ablate.py Box-2D9P 8192x8192 -1 $m 4 > /dev/null 2>&1
  ncu -i gpurun_out/h16j/m$m.ncu-rep --page details > gpurun_out/h16j/details_m$m.txt 2>&1
  ncu -i gpurun_out/h16j/m$m.ncu-rep --page raw --csv > gpurun_out/h16j/raw_m$m.csv 2>&1
done
SST_H16=0 SST_DEBUG_MODE=7 timeout 300 ncu --set full --clock-control none -k regex:stencil_step -s 6 -c 1 -o gpurun_out/h16j/f32m7 python tools/ablate.py Box-2D9P 8192x8192 -1 7 4 > /dev/null 2>&1
ncu -i gpurun_out/h16j/f32m7.ncu-rep --page details > gpurun_out/h16j/details_f32m7.txt 2>&1
ncu -i gpurun_out/h16j/f32m7.ncu-rep --page raw --csv > gpurun_out/h16j/raw_f32m7.csv 2>&1
rm -f gpurun_out/h16j/*.ncu-rep
