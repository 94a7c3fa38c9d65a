# Determinism of the default build while another process time-slices the GPU.
export CUDA_MODULE_LOADING=EAGER
python tools/dbg_timeslice.py ref /tmp/ref_default.npy
(timeout 500 python tools/dbg_timeslice.py check /tmp/ref_default.npy 1000 > gpurun_out/r02w_ts_loader.log 2>&1 &)
sleep 10
timeout 400 python tools/dbg_timeslice.py check /tmp/ref_default.npy 8 > gpurun_out/r02w_ts_default.log 2>&1
