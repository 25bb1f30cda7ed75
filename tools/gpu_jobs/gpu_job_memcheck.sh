# compute-sanitizer memcheck over tools/sanitize_cases.py (one tool per gpurun call)
timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo plain_rc=$?
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_cases.py > gpurun_out/san_memcheck.log 2>&1; echo memcheck_rc=$?
tail -5 gpurun_out/san_memcheck.log
