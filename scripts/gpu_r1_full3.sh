set -x
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/t_full3.log 2>&1; echo tests rc=$?
