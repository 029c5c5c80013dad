# GPU round check: full GPU test suite (incl. the slow scale tests) + one bench line.
# usage (from the repo root, on a gpurun box): bash scripts/gpu_tests.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
lscpu > gpurun_out/lscpu_$TAG.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/pytest_gpu_$TAG.txt 2>&1
tail -5 gpurun_out/pytest_gpu_$TAG.txt
