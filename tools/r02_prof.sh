# round-2 profile pass: smoke, bench line (+ reference arm), launch list, ncu --set full of
# both solver kernels, panel trace.  Usage: bash tools/r02_prof.sh TAG
T=${1:-r02}
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo rc=$? >> gpurun_out/smoke_$T.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:chol_tc_kernel -s 1 -c 1 -o gpurun_out/solver_$T -f \
    python tools/prof_solver.py --reps 2 > gpurun_out/ncu_solver_$T.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:chol_backsub -s 1 -c 1 -o gpurun_out/backsub_$T -f \
    python tools/prof_solver.py --reps 2 > gpurun_out/ncu_backsub_$T.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:proj_pair -s 2 -c 1 -o gpurun_out/proj_$T -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_proj_$T.log 2>&1
if [ -f paper_2604_10377_b200/libfmap_cuda_t.so ]; then
  FMAP_LIB_VARIANT=t FMAP_TRACE_FILE=gpurun_out/trace_$T.bin FMAP_TRACE_BLOCK=5 python tools/prof_solver.py --reps 2 > /dev/null 2>&1
  python tools/trace_panel.py gpurun_out/trace_$T.bin > gpurun_out/trace_panel_$T.txt 2>&1
fi
