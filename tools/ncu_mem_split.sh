M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_sector_op_write_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__d_sectors_fill_sysmem.sum,lts__d_sectors_fill_device.sum,lts__t_sectors_srcunit_ltcfabric.sum
mkdir -p gpurun_out/tr
for m in 0 16 32 6; do
  SST_VARIANT=10 SST_DEBUG_MODE=$m timeout 300 ncu --metrics $M --clock-control none -k regex:stencil -s 4 -c 1 --csv python tools/ablate.py Box-3D27P 512x512x512 10 $m 4 > gpurun_out/tr/ncu3d_m$m.csv 2>&1
done
SST_DEBUG_MODE=0 timeout 300 ncu --metrics $M --clock-control none -k regex:stencil -s 4 -c 1 --csv python tools/ablate.py Box-2D9P 8192x8192 -1 0 4 > gpurun_out/tr/ncu2d_m0.csv 2>&1
SST_DEBUG_MODE=1 timeout 300 ncu --metrics $M --clock-control none -k regex:stencil -s 4 -c 1 --csv python tools/ablate.py Box-2D9P 8192x8192 -1 1 4 > gpurun_out/tr/ncu2d_m1.csv 2>&1
