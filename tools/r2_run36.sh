# round-2 GPU session 36 (final code): full GPU suite, smoke, bench + reference arm, ncu launch list / traffic, full-size config-3 parity
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf --durations=8 > gpurun_out/r2s36_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s36_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2s36_smoke.log 2>&1; echo EXIT $? >> gpurun_out/r2s36_smoke.log
timeout 900 python bench.py > gpurun_out/r2s36_bench.json 2> gpurun_out/r2s36_bench.err; echo EXIT $? >> gpurun_out/r2s36_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2s36_bench_ref.json 2> gpurun_out/r2s36_bench_ref.err; echo EXIT $? >> gpurun_out/r2s36_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2s36_c3_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2s36_ncu_launch.log 2>&1
timeout 2400 python tests/fullsize_parity.py --config c3 --out gpurun_out/r2s36_fullsize_c3.json > gpurun_out/r2s36_fullsize_c3.log 2>&1; echo EXIT $? >> gpurun_out/r2s36_fullsize_c3.log
echo done
