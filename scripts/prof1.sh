set -x
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/p1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_leafs|k_scatter" -s 3 -c 3 \
    -o gpurun_out/p1_c5 -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/p1_ncu.log 2>&1
echo "rc=$?"
