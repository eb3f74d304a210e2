python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
python tools/prof_solver.py --reps 5 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg -k regex:chol_tc -c 2 --clock-control none python tools/prof_solver.py --reps 2 > gpurun_out/ncu_tc.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_tc.log
