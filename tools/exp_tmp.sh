timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 300 python tools/ablate.py Box-3D27P 512x512x512 9,11 0,32 50
timeout 300 python tools/ablate.py Box-2D9P 8192x8192 -1 0 1000
timeout 300 python tools/ablate.py Star-2D13P 16384x16384 -1 0 100
