# ncu --set full of the all-communities table/list kernels (LJ shape, 10 000 communities)
mkdir -p gpurun_out
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_sp_lists" -c 7 -o /tmp/sp_full \
  python tools/sparse_time.py lj 10000 > gpurun_out/sp_ncu.log 2>&1
python tools/ncu_summary.py /tmp/sp_full.ncu-rep > gpurun_out/sp_full_summary.txt
cat gpurun_out/sp_full_summary.txt
