# round-2 GPU session 4: fp64 pipe probe, C-ABI fit tests, bench + reference arm, ncu launch list
cd $GRAFT_REPO_ROOT
timeout 120 ./build/fp64_mix > gpurun_out/r2_fp64_mix.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fit_abi.py tests/test_gpu_rsvd_abi.py -q -x -p no:cacheprovider > gpurun_out/r2_fit_abi.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.log
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_c3_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2_ncu_launch.log 2>&1
echo done
