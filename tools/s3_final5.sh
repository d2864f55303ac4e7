cd $GRAFT_REPO_ROOT
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_bf16 -c 1 -o gpurun_out/s3_final_attn python tools/ncu_steady.py 1500 > gpurun_out/s3_final_ncu_attn.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/s3_final_ncu_attn.log
