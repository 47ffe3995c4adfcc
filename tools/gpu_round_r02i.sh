bash tools/gpu_round2b.sh r02i > gpurun_out/round2b_r02i.log 2>&1
bash tools/gpu_prof_r02.sh r02i > gpurun_out/prof_r02i.log 2>&1
cat gpurun_out/round2b_r02i.log | tail -12
tail -n 3 gpurun_out/sanitizer_*.log
