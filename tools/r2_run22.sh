# round-2 GPU session 22: projection-from-Gram route — full GPU suite, bench, full-size config-3 parity
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf --durations=8 > gpurun_out/r2s22_gputest.log 2>&1; echo EXIT $? >> gpurun_out/r2s22_gputest.log
timeout 900 python bench.py > gpurun_out/r2s22_bench.json 2> gpurun_out/r2s22_bench.err; echo EXIT $? >> gpurun_out/r2s22_bench.err
timeout 2400 python tests/fullsize_parity.py --config c3 --out gpurun_out/r2s22_fullsize_c3.json > gpurun_out/r2s22_fullsize_c3.log 2>&1; echo EXIT $? >> gpurun_out/r2s22_fullsize_c3.log
echo done
