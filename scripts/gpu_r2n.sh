mkdir -p gpurun_out/r2n
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/r2n/pytest_gpu.txt 2>&1; tail -4 gpurun_out/r2n/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/r2n/bench.json 2> gpurun_out/r2n/bench.err; tail -c 200 gpurun_out/r2n/bench.json; tail -3 gpurun_out/r2n/bench.err
