mkdir -p gpurun_out/r02t
timeout 900 python -m pytest tests/test_surface_gpu.py -x -q -s > gpurun_out/r02t/surface.log 2>&1; echo "surface exit $?" >> gpurun_out/r02t/status
bash tools/gpu_prof_agg.sh r02t
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02t/bench_c5.json 2> gpurun_out/r02t/bench_c5.err; echo "bench c5 exit $?" >> gpurun_out/r02t/status
timeout 1500 python -m pytest tests -m gpu -q -x -k "aggregat or determin or composite or c3_reduced or shell or c5" > gpurun_out/r02t/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02t/status
