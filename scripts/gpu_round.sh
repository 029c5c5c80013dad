# One GPU round check: GPU tests, a bench line, optional ncu launch list.
# usage (on a gpurun box, from the repo root): bash scripts/gpu_round.sh TAG [ncu]
TAG=${1:-run}
mkdir -p gpurun_out
bash scripts/gpu_tests.sh $TAG
bash scripts/gpu_bench.sh $TAG
if [ "$2" = "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-extra --no-cpu > gpurun_out/ncu_bench_$TAG.log 2>&1
fi
