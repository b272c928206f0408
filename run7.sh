for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_stress.py -x -q > gpurun_out/fev3_stress_$i.log 2>&1; echo stress rc $?; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_fill_async.py tests/test_gpu_plugin.py tests/test_gpu_policies.py -x -q -k "not full_1m" > gpurun_out/fev3_tests.log 2>&1; echo tests rc $?
timeout 300 python bench.py --no-cpu --no-sub --steps 20 > gpurun_out/fev3_bench.json 2> gpurun_out/fev3_bench.err; echo bench rc $?
timeout 300 python bench.py --no-cpu --no-sub --steps 20 --workload c2 > gpurun_out/fev3_bench_c2.json 2> gpurun_out/fev3_bench_c2.err; echo bench c2 rc $?
