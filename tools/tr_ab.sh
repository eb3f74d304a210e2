for v in t t2; do
FMAP_LIB_VARIANT=$v FMAP_TRACE_FILE=gpurun_out/trace_$v.bin FMAP_TRACE_BLOCK=5 python tools/prof_solver.py --reps 2 > /dev/null 2>&1
python tools/trace_panel.py gpurun_out/trace_$v.bin | head -30 > gpurun_out/trace_$v.txt
done
