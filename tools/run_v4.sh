bash tools/gpu_srcprof.sh pe '^k_phase_e$' 1
python tools/ncu_world.py --world 8 > gpurun_out/w8_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/w8_launches.csv python tools/ncu_world.py --world 8 > gpurun_out/w8_ncu.log 2>&1
ls -la gpurun_out | grep -E 'pe_|w8_'
