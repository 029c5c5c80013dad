# full ncu capture of selected kernels: KERNELS="regex1 regex2" bash scripts/ncu_one.sh
set -x
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-extra"
for K in $KERNELS; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K $B > gpurun_out/ncu_$K.log 2>&1
done
ls -la gpurun_out
