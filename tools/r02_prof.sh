# round-2 profile pass: bench line, launch list, ncu --set full of both solver kernels, panel trace
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:chol_tc_kernel -s 1 -c 1 -o gpurun_out/solver_r02 -f \
    python tools/prof_solver.py --reps 2 > gpurun_out/ncu_solver.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:chol_backsub -s 1 -c 1 -o gpurun_out/backsub_r02 -f \
    python tools/prof_solver.py --reps 2 > gpurun_out/ncu_backsub.log 2>&1
FMAP_LIB_VARIANT=t FMAP_TRACE_FILE=gpurun_out/trace.bin FMAP_TRACE_BLOCK=5 python tools/prof_solver.py --reps 2 > gpurun_out/trace_run.log 2>&1
python tools/trace_panel.py gpurun_out/trace.bin > gpurun_out/trace_panel.txt 2>&1
python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1
