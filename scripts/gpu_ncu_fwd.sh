set -x
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moba_fwd_ts -s 2 -c 1 -o gpurun_out/prof_fwd_ts python scripts/run_fwd_once.py > gpurun_out/ncu_fwd_ts.log 2>&1
tail -3 gpurun_out/ncu_fwd_ts.log
