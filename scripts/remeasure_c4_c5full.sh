mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/f_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/f_tests.log
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/m_bench_C4.json 2> gpurun_out/m_bench_C4.err; echo "bench C4 rc=$?"
python bench.py --config C4 --steps 2 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_plain_C4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/m_c4_launches.csv python bench.py --config C4 --steps 2 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_ncu_launch_C4.log 2>&1; echo "launch C4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_leafs" -s 6 -c 4 \
    -o gpurun_out/m_c5_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_ncu_c5.log 2>&1; echo "c5 full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_block_tiles|k_block_bounds" -s 2 -c 2 \
    -o gpurun_out/m_c4_full -f python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_ncu_c4.log 2>&1; echo "c4 full rc=$?"
