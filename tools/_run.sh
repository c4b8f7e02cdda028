mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; tail -3 gpurun_out/pytest_gpu2.log
timeout 600 python tools/synth_perf.py --config 3 --reps 3 --paths "v2;direct_hot" > gpurun_out/synth3j.log 2>&1; cat gpurun_out/synth3j.log | cut -c1-200
timeout 1500 python bench.py --config 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench_rc=$?; cat gpurun_out/bench3.json
