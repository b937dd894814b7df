# round-2 GPU session 20: projection from the snapshot Gram — GPU suite + bench
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x --durations=8 > gpurun_out/r2s20_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s20_gputest.log
timeout 900 python bench.py > gpurun_out/r2s20_bench.json 2> gpurun_out/r2s20_bench.err; echo EXIT $? >> gpurun_out/r2s20_bench.err
echo done
