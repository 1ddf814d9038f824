#!/bin/bash
# One GPU session of round-end evidence (run under gpurun from the repo root):
# GPU tests, the bench line, the bench's ncu launch list, ncu --set full
# captures of the dominant product kernel of each config, the per-config
# lambda-vs-BB table and the approach-from-below table.  Outputs land in
# gpurun_out/ and are copied into profiles/ on the dev box.
set -u
R=${1:-r01}
O=gpurun_out
mkdir -p $O
python -m pytest tests -q -m gpu > $O/${R}_gpu_tests.log 2>&1; tail -2 $O/${R}_gpu_tests.log
python bench.py > $O/${R}_bench.jsonl 2> $O/${R}_bench.err; tail -c 300 $O/${R}_bench.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${R}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
FULL="ncu --set full --clock-control none --import-source on"
$FULL -k regex:k_tile2 -s 2 -c 1 -o $O/${R}_edm_c2 -f \
    python scripts/one.py --m 2 --n 65536 --payload edm --rho 256 --gran tile --layout tiles --flags 4 --reps 3 > /dev/null 2>&1
$FULL -k regex:k_tile3 -s 2 -c 1 -o $O/${R}_iwa_c3 -f \
    python scripts/one.py --m 3 --n 1024 --payload index_write_atm --param 0.01 --rho 32 --gran tile --layout tiles --flags 4 --reps 3 > /dev/null 2>&1
$FULL -k regex:k_tile3 -s 2 -c 1 -o $O/${R}_iw_c3 -f \
    python scripts/one.py --m 3 --n 1024 --payload index_write --rho 32 --gran tile --layout tiles --flags 4 --reps 3 > /dev/null 2>&1
$FULL -k regex:k_tile3 -s 2 -c 1 -o $O/${R}_atm_c3 -f \
    python scripts/one.py --m 3 --n 1024 --payload atm --param 0.01 --rho 32 --gran tile --reps 3 > /dev/null 2>&1
$FULL -k regex:k_tile3 -s 2 -c 1 -o $O/${R}_tc_c5 -f \
    python scripts/one.py --m 3 --n 2048 --payload tc --param 0.5 --rho 64 --gran tile --persistent 32 --reps 3 > /dev/null 2>&1
$FULL -k regex:k_tile2 -s 2 -c 1 -o $O/${R}_iw_c4 -f \
    python scripts/one.py --m 2 --n 131072 --payload index_write --rho 128 --gran tile --layout tiles --flags 4 --reps 3 > /dev/null 2>&1
python scripts/configs_bench.py > $O/${R}_configs.log 2>&1
cp $O/configs.json $O/${R}_configs.json 2>/dev/null
python scripts/below_bench.py > $O/${R}_below.log 2>&1
cp $O/below.json $O/${R}_below_vs_above.json 2>/dev/null
python scripts/shard_emulation.py > $O/${R}_shards.log 2>&1
cp $O/shards.json $O/${R}_shard_emulation.json 2>/dev/null
python scripts/sustained.py > $O/${R}_sustained.log 2>&1
cp $O/sustained.json $O/${R}_sustained_power_cap.json 2>/dev/null
# summaries here (ncu is on the box); the large reports stay behind (gpurun_out <= 64 MiB)
for k in edm_c2 iwa_c3 iw_c3 atm_c3 tc_c5 iw_c4; do
    python scripts/ncu_summary.py $O/${R}_$k.ncu-rep $O/${R}_${k}_ncu_full.json > /dev/null 2>&1
done
rm -f $O/${R}_*.ncu-rep
ls -la $O | tail -30
