# round-2 GPU session 17: double-buffered TMA-store epilogue vs register stores (interleaved grid)
cd $GRAFT_REPO_ROOT
FDMD_TC2_TMAO=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "tc_decode" > gpurun_out/r2_tmao2_tests.log 2>&1
timeout 600 python tools/prof_tc.py --batches 256 512 > gpurun_out/r2_prof_tc_il.txt 2>&1
FDMD_TC2_TMAO=1 timeout 600 python tools/prof_tc.py --batches 256 512 > gpurun_out/r2_prof_tc_il_tmao.txt 2>&1
echo done
