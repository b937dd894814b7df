# round-2 GPU session 9: 5x9 panel tiles + periodic fragment offsets (tests, sweep), C-ABI DMDc test, power limits
cd $GRAFT_REPO_ROOT
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE > gpurun_out/r2_smi_power.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "gram" > gpurun_out/r2_gram_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fit_abi.py -q -p no:cacheprovider > gpurun_out/r2_fit_abi.log 2>&1
timeout 600 python tools/gram_sweep.py --splits 0 > gpurun_out/r2_gram_sweep_w9.txt 2>&1
FDMD_GRAM_WC=7 timeout 600 python tools/gram_sweep.py --splits 0 > gpurun_out/r2_gram_sweep_w7.txt 2>&1
echo done
