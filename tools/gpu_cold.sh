timeout 300 python tools/cold_setup_probe.py c5 2>&1 | tee gpurun_out/cold_setup.txt
CUDA_MODULE_LOADING=EAGER timeout 300 python tools/cold_setup_probe.py c5 2>&1 | tee -a gpurun_out/cold_setup.txt
timeout 300 python tools/cold_setup_probe.py c4 2>&1 | tee -a gpurun_out/cold_setup.txt
