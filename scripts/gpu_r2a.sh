# round-2 first GPU pass: GPU test suite, smoke, default bench line
mkdir -p gpurun_out/r2a
nvidia-smi -L > gpurun_out/r2a/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 600 > gpurun_out/r2a/pytest_gpu.txt 2>&1; tail -3 gpurun_out/r2a/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.txt 2>&1; tail -2 gpurun_out/r2a/smoke.txt
timeout 900 python bench.py > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err; tail -c 600 gpurun_out/r2a/bench.json; tail -5 gpurun_out/r2a/bench.err
