mkdir -p gpurun_out
CMD="python scripts/chain_check.py 128 6 /tmp/zc.npy"
$CMD > gpurun_out/chain_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 2 -c 2 -o gpurun_out/prof_chain $CMD > gpurun_out/ncu_chain.log 2>&1; echo ncu=$?
