# one traced cfg2 solve (CTA 5, its second system) -> per-panel breakdown
FMAP_TRACE_FILE=gpurun_out/trace.bin FMAP_TRACE_BLOCK=5 python tools/prof_solver.py --reps 2 > gpurun_out/trace_run.log 2>&1
python tools/trace_panel.py gpurun_out/trace.bin > gpurun_out/trace_panel.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/gputest8.log 2>&1; echo rc=$? >> gpurun_out/gputest8.log
