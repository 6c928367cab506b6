mkdir -p gpurun_out/r02v
timeout 300 python tools/peaks.py gpurun_out/r02v/peaks.json > gpurun_out/r02v/peaks.log 2>&1; echo "peaks exit $?" >> gpurun_out/r02v/status
bash tools/gpu_prof_agg.sh r02v
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02v/bench_c5.json 2> gpurun_out/r02v/bench_c5.err; echo "bench c5 exit $?" >> gpurun_out/r02v/status
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_coarsen|k_hist|k_scatter' --csv --log-file gpurun_out/r02v/launches_c5.csv python tools/profile_frame.py --config 5 --frames 1 > gpurun_out/r02v/ncu_l.log 2>&1; echo "launch exit $?" >> gpurun_out/r02v/status
timeout 900 python bench.py --config 6 --steps 5 --warmup 3 > gpurun_out/r02v/bench_c6.json 2> gpurun_out/r02v/bench_c6.err; echo "bench c6 exit $?" >> gpurun_out/r02v/status
timeout 1500 python -m pytest tests -m gpu -q -x -k "aggregat or determin or c5 or surface or composite" > gpurun_out/r02v/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02v/status
