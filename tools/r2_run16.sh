# round-2 GPU session 16: tc_decode2 grid with interleaved frame tiles (L2 sharing of basis rows)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "planes or tc_decode" > gpurun_out/r2_il_tests.log 2>&1
timeout 600 python tools/prof_tc.py --batches 256 512 > gpurun_out/r2_prof_tc_il.txt 2>&1
FDMD_TC2_TMAO=1 timeout 600 python tools/prof_tc.py --batches 256 512 > gpurun_out/r2_prof_tc_il_tmao.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tc_decode2 --csv --log-file gpurun_out/r2_il_launches.csv python tools/prof_tc.py --batches 512 > /dev/null 2>&1
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2_bench_il.json 2> gpurun_out/r2_bench_il.log
echo done
