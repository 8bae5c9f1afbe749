# batch 32, every bench layer, TF32 + BF16 (fp32 activations): the full knob
# space + forced K split 2, on the current library (re-derives the batch-32 records)
A="--batch 32 --which all --splits 2"
python tools/tune_ncu.py --profile-pass $A --out gpurun_out/tune_b32_launches.json > gpurun_out/tune_b32_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    -k 'regex:tc_gemm|exact_gemm|tail_reduce|splitk_reduce|pack_filter|to_bf16|pointwise_gather|split3|pad_phase' --csv --log-file gpurun_out/tune_b32_ncu.csv \
    python tools/tune_ncu.py --profile-pass $A --out gpurun_out/tune_b32_launches.json > gpurun_out/tune_b32_ncu.log 2>&1
echo DONE $?
