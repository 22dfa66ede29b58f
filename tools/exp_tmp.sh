FLUSH=2 SST_MULTISTEP=0 timeout 300 python tools/ablate.py Box-2D9P 4096x4096 0,2 0 100
SST_MULTISTEP=0 timeout 300 python tools/ablate.py Heat-2D 8192x8192 0,2 0 200
SST_MULTISTEP=0 timeout 300 python tools/ablate.py Box-2D9P 8192x8192 0,2 0 200
timeout 300 python tools/ablate.py Heat-2D 8192x8192 0,2 0 200
timeout 300 python tools/ablate.py Box-2D9P 8192x8192 0,2 0 200
