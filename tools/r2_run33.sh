# round-2 GPU session 33: svd(B) through cuSOLVER gesvdp (fdmd_svd_small) — kernel test, parity suites, bench
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py tests/test_gpu_config2.py tests/test_gpu_sharded.py tests/test_gpu_cli.py tests/test_gpu_model_io.py tests/test_gpu_serving.py -q --timeout 900 -p no:cacheprovider -rf --durations=5 > gpurun_out/r2s33_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s33_gputest.log
timeout 900 python bench.py > gpurun_out/r2s33_bench.json 2> gpurun_out/r2s33_bench.err; echo EXIT $? >> gpurun_out/r2s33_bench.err
echo done
