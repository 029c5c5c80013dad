# forward change check: GPU tests, timelines at C2 / 64K, stage split
mkdir -p gpurun_out
TAG=${1:-f}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_$TAG.txt
ROWS=40 timeout 300 python scripts/trace_fwd.py > gpurun_out/trace_fwd_c2_$TAG.txt 2>&1; tail -2 gpurun_out/trace_fwd_c2_$TAG.txt
CFG=32,65536,64,128,8 ROWS=40 timeout 300 python scripts/trace_fwd.py > gpurun_out/trace_fwd_64k_$TAG.txt 2>&1; tail -2 gpurun_out/trace_fwd_64k_$TAG.txt
timeout 600 python scripts/stage_split.py C2 64K C4 > gpurun_out/stages_$TAG.txt 2>&1; cat gpurun_out/stages_$TAG.txt
