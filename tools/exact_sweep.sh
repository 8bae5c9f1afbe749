# SGEMM 1024^3 exact FP32: library tile (h,w,r,c) and ring depth sweep
for t in 8,4,8,16 8,8,8,16 4,4,8,16 4,4,16,16 4,8,16,8 8,4,16,16 4,4,16,8 2,4,16,16 4,2,16,16 8,2,16,16 2,8,16,16 4,4,8,8; do
  for st in 2 3; do
    echo -n "tile=$t stages=$st: "
    TK_EXPERIMENTS=1 TK_EXACT_TILE=$t TK_EXACT_STAGES=$st python tools/sgemm_probe.py 1024 2>&1 | grep 'fp32' | head -1
  done
done
