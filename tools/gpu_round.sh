mkdir -p gpurun_out
python tools/shape_sweep.py > gpurun_out/shape_sweep.md 2> gpurun_out/shape_sweep.err
