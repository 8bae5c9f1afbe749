# VGG16 at batch 32 in 3xTF32 (bench.py's vgg16_3xtf32 leg)
A="--batch 32 --which vgg16 --precisions 3xtf32 --splits 2"
python tools/tune_ncu.py --profile-pass $A --out gpurun_out/tune_3x_launches.json > gpurun_out/tune_3x_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    -k 'regex:tc_gemm|exact_gemm|tail_reduce|splitk_reduce|pack_filter|to_bf16|pointwise_gather|split3|pad_phase' --csv --log-file gpurun_out/tune_3x_ncu.csv \
    python tools/tune_ncu.py --profile-pass $A --out gpurun_out/tune_3x_launches.json > gpurun_out/tune_3x_ncu.log 2>&1
echo DONE $?
