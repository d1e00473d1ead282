timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; cat gpurun_out/bench4.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:partition --csv python tools/plan_once.py cfg4 1 2>&1 | grep -i duration | tail -2
