# round-2 GPU session 27: tc_decode2 staged epilogue with 16-byte stores (FDMD_TC2_TMAO=2) vs register stores
cd $GRAFT_REPO_ROOT
FDMD_TC2_TMAO=2 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q --timeout 300 -p no:cacheprovider -rf -k "tc_decode or config3_config4 or reconstruct" > gpurun_out/r2s27_tests_m2.log 2>&1; echo EXIT $? >> gpurun_out/r2s27_tests_m2.log
timeout 300 python tools/prof_tc.py --batches 256 512 > gpurun_out/r2s27_prof_m0.txt 2>&1
FDMD_TC2_TMAO=2 timeout 300 python tools/prof_tc.py --batches 256 512 > gpurun_out/r2s27_prof_m2.txt 2>&1
FDMD_TC2_TMAO=1 timeout 300 python tools/prof_tc.py --batches 256 512 > gpurun_out/r2s27_prof_m1.txt 2>&1
echo done
