#!/bin/bash
# End-of-milestone measurement on one B200 (gpurun): gpu tests, one bench line per
# BASELINE config (with e2e and the CPU-oracle baselines), every config's ncu launch list
# (kernel times + DRAM bytes: the per-marker traffic bench.py reports) and full ncu
# captures of the dominant kernels of C5 and C4.  Outputs under gpurun_out/.
# usage: bash scripts/round_measure.sh [notests]
mkdir -p gpurun_out
if [ "$1" != "notests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/m_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/m_tests.log
fi
for c in C5 C4 C3a C3b C2a C2b C1; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/m_bench_$c.json 2> gpurun_out/m_bench_$c.err
  echo "bench $c rc=$?"
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/m_ref_C5.json 2> gpurun_out/m_ref_C5.err; echo "ref rc=$?"
for c in C5 C4 C3a C3b C2a C2b C1; do
  lc=$(echo $c | tr A-Z a-z)
  python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/m_${lc}_launches.csv python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_ncu_launch_$c.log 2>&1
  echo "launches $c rc=$?"
done
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_plain_full5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_leafs" -s 6 -c 4 \
    -o gpurun_out/m_c5_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_ncu_c5.log 2>&1
echo "c5 full rc=$?"
python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_plain_full4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_block_tiles|k_block_bounds" -s 2 -c 2 \
    -o gpurun_out/m_c4_full -f python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_ncu_c4.log 2>&1
echo "c4 full rc=$?"
python benchmarks/table2.py --reps 5 --out gpurun_out/m_table2.md > gpurun_out/m_table2.log 2>&1; echo "table2 rc=$?"
