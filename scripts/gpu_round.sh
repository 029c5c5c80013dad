set -x
timeout 900 python bench.py > gpurun_out/bench_s6.json 2> gpurun_out/bench_s6.err; tail -2 gpurun_out/bench_s6.err; cat gpurun_out/bench_s6.json
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s6.txt 2>&1; tail -2 gpurun_out/pytest_gpu_s6.txt
KERNELS="moba_bwd_pipe moba_fwd_ts route_topk_tc2 moba_combine varlen_scatter centroid_warp bwd_preprocess" timeout 1200 bash scripts/ncu_profile.sh > /dev/null 2>&1
ls gpurun_out
