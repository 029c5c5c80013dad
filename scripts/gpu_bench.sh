# bench line + reference arm on the GPU box: bash scripts/gpu_bench.sh TAG [bench args]
TAG=${1:-run}; shift
mkdir -p gpurun_out
timeout 1500 python bench.py "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err; cut -c1-600 gpurun_out/bench_$TAG.json
