# round-2 GPU session 29: side lines with stage traces (config 2 DMDc, config 1 exact DMD as BASELINE writes it)
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config c2 > gpurun_out/r2s29_bench_c2.json 2> gpurun_out/r2s29_bench_c2.err; echo EXIT $? >> gpurun_out/r2s29_bench_c2.err
timeout 600 python bench.py --config c1x > gpurun_out/r2s29_bench_c1x.json 2> gpurun_out/r2s29_bench_c1x.err; echo EXIT $? >> gpurun_out/r2s29_bench_c1x.err
echo done
