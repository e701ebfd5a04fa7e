# launch list of the all-communities mode (LJ shape, 10 000 communities), run on the GPU box
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 200 --csv \
  --log-file gpurun_out/sparse_l.csv python tools/sparse_time.py lj 10000 > /dev/null 2>&1
python tools/launches.py gpurun_out/sparse_l.csv 25
