# round-2 GPU session 11: plane-output lift tests, bench (planes schedule), ncu full of the 512-frame reconstruct
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q -p no:cacheprovider -k "planes or tc_decode or config3_config4 or tcgen05_lift" > gpurun_out/r2_planes_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench_c3_p.json 2> gpurun_out/r2_bench_c3_p.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_decode2 -c 1 -o gpurun_out/r2_tc2_b512 python tools/prof_tc.py --batches 512 > gpurun_out/r2_ncu_tc2.log 2>&1
echo done
