# GPU check of the round-2 changes: new tests first, then the whole GPU suite, then a quick bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_baseline_configs.py tests/test_gpu_pipeline.py -m gpu -x -q -k "config or density or gaussian_size or sparse_batch or multi_iteration" > gpurun_out/pytest_new.log 2>&1; echo "rc $?" >> gpurun_out/pytest_new.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1
