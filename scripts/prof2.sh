set -x
python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/p2_plain.json 2>gpurun_out/p2_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:"k_leafs|k_scatter" -s 3 -c 3 \
    -o gpurun_out/p2_c5 -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/p2_ncu.log 2>&1
echo "rc=$?"
