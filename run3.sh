timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gputests_r02a.log 2>&1; echo tests rc $?
timeout 600 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo bench rc $?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r02a.json 2> gpurun_out/bench_ref_r02a.err; echo ref rc $?
