# round-2 GPU session 7: C-ABI tests (ldq fix, Householder fallback), cluster Gram w/ relaxed arrives, bench diag
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fit_abi.py tests/test_gpu_rsvd_abi.py -q -p no:cacheprovider > gpurun_out/r2_fit_abi.log 2>&1
timeout 300 python tools/dbg_dmdc.py > gpurun_out/r2_dbg_dmdc.txt 2>&1
timeout 600 python tools/gram_sweep.py --splits 0 > gpurun_out/r2_gram_sweep_cl2.txt 2>&1
FDMD_GRAM_CLUSTER=0 FDMD_BENCH_DIAG=1 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2_bench_diag.json 2> gpurun_out/r2_bench_diag.log
echo done
