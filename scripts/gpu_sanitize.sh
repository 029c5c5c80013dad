# compute-sanitizer over every hot-path kernel at small shapes (scripts/sanitize_run.py)
mkdir -p gpurun_out
for T in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 50 python scripts/sanitize_run.py > gpurun_out/sanitize_$T.txt 2>&1
  echo "$T rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$T.txt >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
