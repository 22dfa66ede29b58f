timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/memcheck.log 2>&1; tail -15 gpurun_out/memcheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/synccheck.log 2>&1; tail -8 gpurun_out/synccheck.log
