# final evidence on one box: GPU tests, bench line, ncu launch list + captures
TAG=${1:-r02f}
mkdir -p gpurun_out
bash scripts/gpu_tests.sh $TAG
bash scripts/gpu_bench.sh $TAG
# compute-sanitizer is closed on the GPU pool (it left GPUs needing a reset);
# scripts/gpu_sanitize.sh is kept for boxes where it is allowed
bash scripts/gpu_ncu_round.sh ${TAG}_64k b2h16_n65536_d64
