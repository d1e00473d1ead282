set -x
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err; cat gpurun_out/bench2.json
for w in cfg1 cfg2 cfg3; do HPK_MINQ=0 timeout 300 python tools/cap_sweep.py $w 256,512,1024; done
