export LCO_MSD=1 LCO_MSD_CTA=1
python scripts/kprof.py C3 0 0,3,1,4,2,5 > gpurun_out/d_c3b.log 2>&1; echo rc=$?
ncu --set full --clock-control none -k regex:"k_leaf<" -c 1 -o gpurun_out/d_c3b -f python scripts/kprof.py C3 0 0,3,1,4,2,5 > gpurun_out/d_c3b_ncu.log 2>&1; echo ncu rc=$?
