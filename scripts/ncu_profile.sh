# ncu evidence for the bench step: launch list + full captures of the top kernels.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-extra"
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > /dev/null 2>&1
for K in ${KERNELS:-moba_bwd_pipe moba_fwd_ts route_tc_kernel moba_combine varlen_scatter centroid_warp bwd_preprocess}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K $B > /dev/null 2>&1
done
ls -la gpurun_out
