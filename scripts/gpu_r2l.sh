mkdir -p gpurun_out/r2l
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/r2l/pytest_gpu.txt 2>&1; tail -4 gpurun_out/r2l/pytest_gpu.txt
timeout 900 python bench.py --no-same-config > gpurun_out/r2l/bench.json 2> gpurun_out/r2l/bench.err; tail -c 300 gpurun_out/r2l/bench.json; tail -3 gpurun_out/r2l/bench.err
