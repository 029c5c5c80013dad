# full ncu capture of the tc router at one shape: bash scripts/ncu_route.sh TAG H N d B k
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_tc_kernel -s 1 -c 1 \
  -o gpurun_out/prof_route_$TAG python scripts/route_probe.py "$@" tc 2 > gpurun_out/ncu_route_$TAG.log 2>&1
tail -2 gpurun_out/ncu_route_$TAG.log
