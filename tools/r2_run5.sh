# round-2 GPU session 5: C-ABI fit tests (incl. DMDc), panel-Gram split sweep at config-3 size
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fit_abi.py -q -p no:cacheprovider > gpurun_out/r2_fit_abi.log 2>&1
timeout 900 python tools/gram_sweep.py > gpurun_out/r2_gram_sweep.txt 2>&1
echo done
