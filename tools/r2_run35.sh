# round-2 GPU session 35: fused pair statistics with f32 magnitudes — kernel test, modes parity, bench
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q --timeout 300 -p no:cacheprovider -rf -k "fused_pair_stats or tc_decode or pair_stats" > gpurun_out/r2s35_kernel.log 2>&1; echo EXIT $? >> gpurun_out/r2s35_kernel.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_sharded.py -q --timeout 600 -p no:cacheprovider -rf > gpurun_out/r2s35_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s35_gputest.log
timeout 900 python bench.py --no-cpu > gpurun_out/r2s35_bench.json 2> gpurun_out/r2s35_bench.err; echo EXIT $? >> gpurun_out/r2s35_bench.err
FDMD_TC_STATS=0 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2s35_bench_nofuse.json 2> gpurun_out/r2s35_bench_nofuse.err; echo EXIT $? >> gpurun_out/r2s35_bench_nofuse.err
echo done
