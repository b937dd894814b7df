# round-2 GPU session 30: span-only eigen fallback for singular sketch Grams — config-2 / DMDc / fallback tests, c2 bench
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_config2.py tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_rsvd_abi.py -q --timeout 600 -p no:cacheprovider -rf --durations=5 > gpurun_out/r2s30_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s30_gputest.log
timeout 600 python bench.py --config c2 > gpurun_out/r2s30_bench_c2.json 2> gpurun_out/r2s30_bench_c2.err; echo EXIT $? >> gpurun_out/r2s30_bench_c2.err
echo done
