DB=profiles/r02_tune_ncu.ndjson,profiles/r02_tune_gemm.ndjson
for p in tf32 bf16; do ./tools/tk_sweep $p gpurun_out/r02_sweep_${p}_tuned.csv all $DB > gpurun_out/sweep_$p.log 2>&1; echo "$p $?"; done
./tools/tk_sweep tf32 gpurun_out/r02_sweep_tf32_rules.csv all > gpurun_out/sweep_tf32_rules.log 2>&1; echo "rules $?"
