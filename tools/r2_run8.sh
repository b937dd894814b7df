# round-2 GPU session 8: DMDc C-ABI debug, XtX after reconstruct (clock/power), cluster Gram with relaxed arrives
cd $GRAFT_REPO_ROOT
timeout 300 python tools/dbg_dmdc.py > gpurun_out/r2_dbg_dmdc.txt 2>&1
timeout 600 python tools/xtx_after_recon.py > gpurun_out/r2_xtx_after_recon.txt 2>&1
timeout 600 python tools/gram_sweep.py --splits 0 > gpurun_out/r2_gram_sweep_cl3.txt 2>&1
echo done
