timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py --workload cfg5 --snapshots 200 --steps 2 --warmup 1 2>gpurun_out/cfg5a.err | tail -1
timeout 900 python bench.py --workload cfg5 --snapshots 1000 --steps 2 --warmup 1 2>gpurun_out/cfg5b.err | tail -1
tail -3 gpurun_out/cfg5b.err
