# round-2 GPU session 26: lift epilogue split in fp32 — planes tests, parity, isolated timing, bench
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py -q --timeout 900 -p no:cacheprovider -rf --durations=5 -k "planes or tall_gemm or parity or config3 or fullsize or optdmd" > gpurun_out/r2s26_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s26_gputest.log
timeout 600 python tools/gram_sweep.py --splits 0 > gpurun_out/r2s26_gram_sweep.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2s26_bench.json 2> gpurun_out/r2s26_bench.err; echo EXIT $? >> gpurun_out/r2s26_bench.err
echo done
