mkdir -p gpurun_out/r02w
timeout 1500 python -m pytest tests -m gpu -q -x -k "aggregat or determin or c5 or c3_reduced or shell" > gpurun_out/r02w/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02w/status
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02w/bench_c5.json 2> gpurun_out/r02w/bench_c5.err; echo "bench c5 exit $?" >> gpurun_out/r02w/status
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_coarsen|k_band|k_hist|k_scatter' --csv --log-file gpurun_out/r02w/launches_c5.csv python tools/profile_frame.py --config 5 --frames 1 > gpurun_out/r02w/ncu_l.log 2>&1; echo "launch exit $?" >> gpurun_out/r02w/status
timeout 900 python bench.py --config 6 --steps 5 --warmup 3 > gpurun_out/r02w/bench_c6.json 2> gpurun_out/r02w/bench_c6.err; echo "bench c6 exit $?" >> gpurun_out/r02w/status
