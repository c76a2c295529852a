#!/bin/bash
# A/B of compile-time variants: bash scripts/variants.sh "<v1 v2 ...>" config...
# (each variants/liblco_<v>.so is copied over the package library in turn)
mkdir -p gpurun_out
vs=$1; shift
cp paper_1802_02619_b200/liblco.so /tmp/liblco_keep.so
for v in $vs; do
  cp variants/liblco_$v.so paper_1802_02619_b200/liblco.so
  for c in "$@"; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/v_${v}_$c.json 2> gpurun_out/v_${v}_$c.err
    echo "$v $c rc=$?"
  done
done
cp /tmp/liblco_keep.so paper_1802_02619_b200/liblco.so
