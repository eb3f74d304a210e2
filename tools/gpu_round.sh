python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
python -m pytest tests -m gpu -x -q > gpurun_out/gputest7.log 2>&1; echo rc=$? >> gpurun_out/gputest7.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo rc=$? >> gpurun_out/bench7.err
