mkdir -p gpurun_out
timeout 1200 python bench.py --config 5 --layout file --no-cpu-baseline --steps 10 > gpurun_out/bench5f.json 2> gpurun_out/bench5f.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench5f.json')); print(d['value'], d['ms_per_step'], d['nonminimal'], d['gate'], d['config']['pilot_layout'])"
timeout 1200 python bench.py --config 5 --no-cpu-baseline --steps 10 > gpurun_out/bench5d.json 2> gpurun_out/bench5d.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench5d.json')); print(d['value'], d['ms_per_step'], d['nonminimal'], d['gate'], d['config']['pilot_layout'])"
