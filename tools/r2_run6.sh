# round-2 GPU session 6: cluster-multicast panel Gram (tests + sweep vs unclustered), DMDc C-ABI debug
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "gram" > gpurun_out/r2_gram_tests.log 2>&1
timeout 600 python tools/gram_sweep.py --splits 0 --after-hbm > gpurun_out/r2_gram_sweep_cl.txt 2>&1
FDMD_GRAM_CLUSTER=0 timeout 600 python tools/gram_sweep.py --splits 0 --after-hbm > gpurun_out/r2_gram_sweep_nocl.txt 2>&1
timeout 300 python tools/dbg_dmdc.py > gpurun_out/r2_dbg_dmdc.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_gram_cl_launches.csv python tools/gram_sweep.py --splits 0 --reps 1 > /dev/null 2>&1
echo done
