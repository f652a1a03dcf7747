# GPU iteration: full gpu test suite (no -x, durations), smoke, bench line.
# Usage: bash scripts/gpu_check.sh [pytest -k expr]
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q ${1:+-k "$1"} --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log
