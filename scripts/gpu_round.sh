set -x
timeout 900 python bench.py > gpurun_out/bench_s12.json 2> gpurun_out/bench_s12.err; tail -2 gpurun_out/bench_s12.err; cat gpurun_out/bench_s12.json
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s12.txt 2>&1; tail -2 gpurun_out/pytest_gpu_s12.txt
KERNELS="moba_bwd_pipe moba_fwd_ts route_topk_tc2 moba_combine varlen_scatter4 centroid_warp bwd_preprocess" timeout 1200 bash scripts/ncu_profile.sh > /dev/null 2>&1
ls gpurun_out
