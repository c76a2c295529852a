#!/bin/bash
# Round-end check on one B200: GPU tests, smoke(), the default bench line, C4 launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/z_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/z_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/z_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/z_smoke.log
timeout 600 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err; echo "bench rc=$?"
python bench.py --config C4 --steps 2 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_plain_C4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/m_c4_launches.csv python bench.py --config C4 --steps 2 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/m_ncu_launch_C4.log 2>&1; echo "launch C4 rc=$?"
