# ncu evidence at the bench workload, summarised on the box (reports stay there)
bash scripts/ncu_profile.sh > gpurun_out/ncu_profile.log 2>&1
python scripts/ncu_summary.py ${1:-r02_64k} ${2:-b2h16_n65536_d64} > gpurun_out/ncu_summary.log 2>&1
cp profiles/${1:-r02_64k}_* profiles/ncu_traffic.json gpurun_out/
for f in gpurun_out/prof_*.ncu-rep; do python scripts/ncu_brief.py $f 30 > ${f%.ncu-rep}.brief.txt 2>&1; done
mkdir -p /tmp/ncu_keep && mv gpurun_out/*.ncu-rep /tmp/ncu_keep/ 2>/dev/null
ls -la gpurun_out
