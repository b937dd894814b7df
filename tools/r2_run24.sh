# round-2 GPU session 24: ncu launch list + traffic of one bench step (projection-from-Gram route), ncu full of
# the dominant kernel (tall_gemm planes lift), c1 / c2 bench lines, full-size config-3 parity
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2s24_c3_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2s24_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tall_gemm_tma -s 1 -c 1 -o gpurun_out/r2s24_tall_gemm_planes python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2s24_ncu_full.log 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/r2s24_bench_c1.json 2> gpurun_out/r2s24_bench_c1.err; echo EXIT $? >> gpurun_out/r2s24_bench_c1.err
timeout 600 python bench.py --config c2 > gpurun_out/r2s24_bench_c2.json 2> gpurun_out/r2s24_bench_c2.err; echo EXIT $? >> gpurun_out/r2s24_bench_c2.err
timeout 2400 python tests/fullsize_parity.py --config c3 --out gpurun_out/r2s24_fullsize_c3.json > gpurun_out/r2s24_fullsize_c3.log 2>&1; echo EXIT $? >> gpurun_out/r2s24_fullsize_c3.log
echo done
