# round-2 GPU session 25: bordered / re-cut panel Gram + tall_gemm K-tail — kernel tests, parity, isolated timings, bench
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_sharded.py tests/test_gpu_fit_abi.py tests/test_gpu_rsvd_abi.py tests/test_gpu_config2.py -q --timeout 900 -p no:cacheprovider -rf --durations=5 > gpurun_out/r2s25_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s25_gputest.log
timeout 600 python tools/gram_sweep.py --splits 0 > gpurun_out/r2s25_gram_sweep.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2s25_bench.json 2> gpurun_out/r2s25_bench.err; echo EXIT $? >> gpurun_out/r2s25_bench.err
echo done
