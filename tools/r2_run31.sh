# round-2 GPU session 31: full-size config-1 parity JSON; functional 2- and 4-rank bench on one GPU (gloo, every rank on cuda:0; timings meaningless)
cd $GRAFT_REPO_ROOT
timeout 900 python tests/fullsize_parity.py --config c1 --out gpurun_out/r2s31_fullsize_c1.json > gpurun_out/r2s31_fullsize_c1.log 2>&1; echo EXIT $? >> gpurun_out/r2s31_fullsize_c1.log
for N in 2 4; do
FDMD_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --config c3s --steps 1 --warmup 1 --no-cpu > gpurun_out/r2s31_bench_c3s_gloo$N.json 2> gpurun_out/r2s31_bench_c3s_gloo$N.err; echo EXIT $? >> gpurun_out/r2s31_bench_c3s_gloo$N.err
done
timeout 600 python bench.py --config c3s --steps 1 --warmup 1 --no-cpu > gpurun_out/r2s31_bench_c3s_1.json 2> gpurun_out/r2s31_bench_c3s_1.err; echo EXIT $? >> gpurun_out/r2s31_bench_c3s_1.err
echo done
