# round-2 GPU session 15: TMA-store frame epilogue for tc_decode2 (tests, prof_tc, bench)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q -p no:cacheprovider -k "planes or tc_decode or config3_config4 or reconstruct or modal" > gpurun_out/r2_tmao_tests.log 2>&1
timeout 600 python tools/prof_tc.py --batches 256 512 > gpurun_out/r2_prof_tc_tmao.txt 2>&1
FDMD_TC2_TMAO=0 timeout 600 python tools/prof_tc.py --batches 256 512 > gpurun_out/r2_prof_tc_regst.txt 2>&1
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2_bench_tmao.json 2> gpurun_out/r2_bench_tmao.log
echo done
