set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -c 2500 gpurun_out/bench.log
