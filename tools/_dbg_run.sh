SLORA_BENCH_TP=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tp1.txt 2> gpurun_out/bench_tp1.err; echo "rc=$?" >> gpurun_out/bench_tp1.err
timeout 300 python -m pytest tests/test_gpu_tp_cabi.py tests/test_gpu_tp.py -q > gpurun_out/tp_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/tp_tests.txt
