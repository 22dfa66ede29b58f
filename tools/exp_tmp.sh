timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for d in 1 0; do SST_DYN=$d FLUSH=2 timeout 300 python tools/ablate.py Heat-2D 4096x4096 -1 0 100; done
timeout 300 python tools/ablate.py Box-2D9P 8192x8192 -1 0 1000
