# round-2 GPU session 19 (re-entry): full GPU test suite + default bench + reference arm
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2s19_smi.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf --durations=15 > gpurun_out/r2s19_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s19_gputest.log
timeout 900 python bench.py > gpurun_out/r2s19_bench.json 2> gpurun_out/r2s19_bench.err; echo EXIT $? >> gpurun_out/r2s19_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2s19_ref.json 2> gpurun_out/r2s19_ref.err
echo done
