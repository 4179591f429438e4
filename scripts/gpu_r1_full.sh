# the round-end checks as the driver runs them: full GPU suite, then smoke()
set -x
time (timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/t_full.log 2>&1); echo tests rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
