# quick GPU check after a kernel change: GPU tests, synccheck + initcheck detail, 64K/512K stage split
TAG=${1:-chk}
mkdir -p gpurun_out
bash scripts/gpu_tests.sh $TAG
timeout 600 compute-sanitizer --tool synccheck python scripts/sanitize_run.py > gpurun_out/sanitize_synccheck_$TAG.txt 2>&1; tail -2 gpurun_out/sanitize_synccheck_$TAG.txt
timeout 900 compute-sanitizer --tool initcheck --print-limit 100000 python scripts/sanitize_run.py > gpurun_out/sanitize_initcheck_$TAG.txt 2>&1; tail -2 gpurun_out/sanitize_initcheck_$TAG.txt
if [ -n "$STAGES" ]; then timeout 900 python scripts/stage_split.py $STAGES > gpurun_out/stages_$TAG.txt 2>&1; tail -20 gpurun_out/stages_$TAG.txt; fi
