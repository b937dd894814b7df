# round-2 GPU session 34: fused pair statistics in the tc_decode2 frame epilogue — kernel test, parity suites, bench
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q --timeout 300 -p no:cacheprovider -rf -k "fused_pair_stats or tc_decode or pair_stats" > gpurun_out/r2s34_kernel.log 2>&1; echo EXIT $? >> gpurun_out/r2s34_kernel.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py tests/test_gpu_cli.py tests/test_gpu_model_io.py -q --timeout 900 -p no:cacheprovider -rf --durations=5 > gpurun_out/r2s34_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s34_gputest.log
timeout 900 python bench.py > gpurun_out/r2s34_bench.json 2> gpurun_out/r2s34_bench.err; echo EXIT $? >> gpurun_out/r2s34_bench.err
echo done
