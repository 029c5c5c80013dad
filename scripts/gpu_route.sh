# router check: bitwise tc == fp32 plans + timings
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_route_tc.py -q -x > gpurun_out/pytest_route.txt 2>&1; tail -5 gpurun_out/pytest_route.txt
for a in "32 8192 64 128 8" "32 65536 64 128 8" "32 524288 64 128 8" "16 65536 128 128 8" "16 524288 128 128 8"; do
  timeout 120 python scripts/route_probe.py $a tc 3 | tail -1
done
timeout 120 python scripts/route_probe.py 32 65536 64 128 8 fp32 2 | tail -1
