set -x
free -g > gpurun_out/free.txt
timeout 1200 python -m pytest tests/test_gpu_cluster_scale.py tests/test_gpu_scale.py -x -q -k "config3 or full_1m" --durations=5 > gpurun_out/parity_new.log 2>&1; echo parity rc $?
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 600 $S --tool $tool --print-limit 40 python -m pytest tests/test_gpu_stress.py -x -q -k "test_random_lockstep[0] or test_random_lockstep[1] or test_random_lockstep[2] or test_random_lockstep[3]" > gpurun_out/san_${tool}_stress.log 2>&1; echo $tool stress rc $?
  timeout 600 $S --tool $tool --print-limit 40 python -m pytest tests/test_gpu_parity.py -x -q -k "example or random-1 or d2lpm" > gpurun_out/san_${tool}_parity.log 2>&1; echo $tool parity rc $?
done
