# round-2 GPU session 21: planes epilogue + border tdot; targeted tests + bench
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_kernels.py -k "planes or tdot" tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py tests/test_gpu_fit_abi.py -q --timeout 900 -p no:cacheprovider -rf --durations=8 > gpurun_out/r2s21_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s21_gputest.log
timeout 900 python bench.py > gpurun_out/r2s21_bench.json 2> gpurun_out/r2s21_bench.err; echo EXIT $? >> gpurun_out/r2s21_bench.err
echo done
