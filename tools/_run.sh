mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; tail -3 gpurun_out/pytest_gpu3.log
timeout 1500 python bench.py --config 4 --no-cpu-baseline --steps 10 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench4.json')); print(d['value'], d['ms_per_step'], d['nonminimal'], d['gate'], d['roofline']['frac'])"
