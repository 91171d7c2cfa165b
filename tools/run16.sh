mkdir -p gpurun_out/r01
timeout 1200 python tools/sweep.py > gpurun_out/r01/sweep_f64.csv 2> gpurun_out/r01/sweep_f64.err
timeout 600 python tools/sweep.py --dtype f32 --fd-n 10 --fd-batches 100000 > gpurun_out/r01/sweep_f32.csv 2> gpurun_out/r01/sweep_f32.err
tail -3 gpurun_out/r01/sweep_f64.err
