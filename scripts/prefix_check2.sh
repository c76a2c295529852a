#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k prefix_plan > gpurun_out/p_newtest.log 2>&1; echo "new test rc=$?"; tail -1 gpurun_out/p_newtest.log
timeout 600 python scripts/ab_prefix.py > gpurun_out/p_ab_new.jsonl 2> gpurun_out/p_ab_new.err; echo "ab new rc=$?"
LCO_NO_PREFIX_MSD=1 timeout 600 python scripts/ab_prefix.py > gpurun_out/p_ab_old.jsonl 2> gpurun_out/p_ab_old.err; echo "ab old rc=$?"
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/p_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/p_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/p_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err; echo "bench rc=$?"
