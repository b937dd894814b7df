# round-2 GPU session 10: compute-sanitizer (memcheck / racecheck / synccheck, one tool per command) + bench
cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --kernel-regex kns=fdmd --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "gram_panel_shapes or tc_decode or pair_stats or test_decode or colmajor or table_apply" > gpurun_out/r2_cs_memcheck_kernels.log 2>&1; echo "exit $?" >> gpurun_out/r2_cs_memcheck_kernels.log
timeout 900 $CS --tool memcheck --kernel-regex kns=fdmd --print-limit 20 python -m pytest tests/test_gpu_fit_abi.py -q -p no:cacheprovider -x -k "small_golden or errors" > gpurun_out/r2_cs_memcheck_fitabi.log 2>&1; echo "exit $?" >> gpurun_out/r2_cs_memcheck_fitabi.log
timeout 1200 $CS --tool racecheck --kernel-regex kns=fdmd --print-limit 20 python -m pytest tests/test_gpu_serving.py -q -p no:cacheprovider -x -k "concurrent" > gpurun_out/r2_cs_racecheck_serving.log 2>&1; echo "exit $?" >> gpurun_out/r2_cs_racecheck_serving.log
FDMD_GRAM_CLUSTER=1 timeout 1200 $CS --tool synccheck --kernel-regex kns=tall_gram_panel --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "gram_panel_shapes" > gpurun_out/r2_cs_synccheck_gram.log 2>&1; echo "exit $?" >> gpurun_out/r2_cs_synccheck_gram.log
timeout 900 python bench.py > gpurun_out/r2_bench_c3_b.json 2> gpurun_out/r2_bench_c3_b.log
echo done
