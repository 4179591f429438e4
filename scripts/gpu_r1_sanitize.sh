set -x
python scripts/sanitize_case.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no python scripts/sanitize_case.py > gpurun_out/san_memcheck.log 2>&1; echo memcheck rc=$?
