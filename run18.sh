timeout 900 python -m pytest tests/test_gpu_stress.py tests/test_gpu_scale.py tests/test_gpu_parity.py -x -q -k "not full_1m" > gpurun_out/k1_tests.log 2>&1; echo tests $?
timeout 300 python bench.py --no-cpu --no-sub --steps 20 > gpurun_out/k1_bench.json 2>&1; echo bench $?
/usr/local/cuda/bin/ncu --set full --clock-control none -k regex:k_match_fast -s 8 -c 1 -o gpurun_out/k1fast2 python bench.py --no-cpu --no-sub --steps 2 --warmup 8 --k1-full-steps 0 > gpurun_out/k1fast2.log 2>&1; echo ncu $?
