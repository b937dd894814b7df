# round-2 GPU session 12: plane tests, HBM write-pattern probe, bench A/B (fp32 basis + split vs planes from the lift)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "planes" > gpurun_out/r2_planes_tests.log 2>&1
timeout 300 ./build/write_pattern > gpurun_out/r2_write_pattern.txt 2>&1
FDMD_BENCH_BASIS=fp32 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2_bench_fp32basis.json 2> gpurun_out/r2_bench_fp32basis.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2_bench_planes.json 2> gpurun_out/r2_bench_planes.log
echo done
