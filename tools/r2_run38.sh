# round-2 GPU session 38: ncu full of the CTA-pair reconstruction (512 frames) and of the modes product with fused statistics
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_decode2 -s 1 -c 1 -o gpurun_out/r2s38_tc2_b512 python tools/prof_tc.py --batches 512 > gpurun_out/r2s38_ncu_tc2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_decode2 -s 3 -c 1 -o gpurun_out/r2s38_tc2_modes_stats python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2s38_ncu_modes.log 2>&1
echo done
