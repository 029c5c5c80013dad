mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_route_tc.py -q -x > gpurun_out/pytest_route.txt 2>&1; tail -3 gpurun_out/pytest_route.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:route_tc_kernel -c 1 -o gpurun_out/prof_rtc64k python scripts/route_probe.py 32 65536 64 128 8 tc 1 > gpurun_out/ncu_rtc64k.log 2>&1
tail -2 gpurun_out/ncu_rtc64k.log
