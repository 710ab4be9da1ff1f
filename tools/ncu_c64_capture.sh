rm -f gpurun_out/ll_c64.txt
QVB200_LAUNCH_LOG=gpurun_out/ll_c64.txt python tools/one_gradient.py 32 4 complex64
IDX=$(awk '$1=="tma"{i++; if ($3==12 && $4>=2 && $5>=32768 && !f) {print i-1; f=1}}' gpurun_out/ll_c64.txt)
echo "idx=$IDX"
ncu --set full --clock-control none --import-source on -k regex:tma_pass -s $IDX -c 1 -o gpurun_out/r02_tma_c64_final python tools/one_gradient.py 32 4 complex64 > gpurun_out/ncu_c64.log 2>&1
echo ncu rc=$?
