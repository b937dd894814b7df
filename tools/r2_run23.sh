# round-2 GPU session 23 (re-entry): projection-from-Gram route — full GPU suite, bench, reference arm
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf --durations=8 > gpurun_out/r2s23_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s23_gputest.log
timeout 900 python bench.py > gpurun_out/r2s23_bench.json 2> gpurun_out/r2s23_bench.err; echo EXIT $? >> gpurun_out/r2s23_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2s23_bench_ref.json 2> gpurun_out/r2s23_bench_ref.err; echo EXIT $? >> gpurun_out/r2s23_bench_ref.err
echo done
