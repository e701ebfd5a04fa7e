# Round profile set (run under gpurun): full bench line, launch list, full ncu
# captures of the Phase E kernels and of the other phases (summarised on the box;
# only the summaries and the Phase E report come back, gpurun_out <= 64 MiB).
# usage: bash tools/gpu_profile.sh TAG
T=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; tail -1 gpurun_out/${T}_bench.log > gpurun_out/${T}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -c 400 --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"^k_phase_e" -c 2 -o gpurun_out/${T}_fullE \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_ncu_fullE.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_fullE.ncu-rep > gpurun_out/${T}_full_phaseE_summary.txt
timeout 900 ncu --set full --clock-control none -k regex:"k_phase_a_|k_phase_d_|k_finalize|k_tk_pass" -c 24 -o /tmp/${T}_fullAD \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_ncu_fullAD.log 2>&1
python tools/ncu_summary.py /tmp/${T}_fullAD.ncu-rep > gpurun_out/${T}_full_phaseAD_summary.txt
ls -la gpurun_out
