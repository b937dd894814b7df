# round-2 GPU session 18: small-solve latency; full GPU test suite
cd $GRAFT_REPO_ROOT
timeout 300 python tools/small_solves.py > gpurun_out/r2_small_solves.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf --durations=10 > gpurun_out/r2_gputest_full.log 2>&1; echo EXIT $? >> gpurun_out/r2_gputest_full.log
echo done
