# final evidence on one box: GPU tests, bench line, sanitizers, ncu launch list + captures
TAG=${1:-r02f}
mkdir -p gpurun_out
bash scripts/gpu_tests.sh $TAG
bash scripts/gpu_bench.sh $TAG
for T in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 100 python scripts/sanitize_run.py > gpurun_out/sanitize_${T}_$TAG.txt 2>&1
  echo "$T rc=$? $(tail -1 gpurun_out/sanitize_${T}_$TAG.txt)"
done
bash scripts/gpu_ncu_round.sh ${TAG}_64k b2h16_n65536_d64
