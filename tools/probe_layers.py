"""Run each ResNet-50 / VGG-16 layer shape once in its own subprocess with a
short timeout (finds hangs / faults without taking the box down)."""
import subprocess
import sys

RES = [("conv1", 7, 2, 224, 3, 64), ("res2a_2a", 1, 1, 56, 64, 64), ("res2a_2b", 3, 1, 56, 64, 64),
       ("res2a_2c", 1, 1, 56, 64, 256), ("res2b_2a", 1, 1, 56, 256, 64), ("res3a_2a", 1, 2, 56, 256, 128),
       ("res3a_2b", 3, 1, 28, 128, 128), ("res3a_2c", 1, 1, 28, 128, 512), ("res3a_1", 1, 2, 56, 256, 512),
       ("res3b_2a", 1, 1, 28, 512, 128), ("res4a_2a", 1, 2, 28, 512, 256), ("res4a_2b", 3, 1, 14, 256, 256),
       ("res4a_2c", 1, 1, 14, 256, 1024), ("res4a_1", 1, 2, 28, 512, 1024), ("res4b_2a", 1, 1, 14, 1024, 256),
       ("res5a_2a", 1, 2, 14, 1024, 512), ("res5a_2b", 3, 1, 7, 512, 512), ("res5a_2c", 1, 1, 7, 512, 2048),
       ("res5a_1", 1, 2, 14, 1024, 2048), ("res5b_2a", 1, 1, 7, 2048, 512)]
batch = sys.argv[1] if len(sys.argv) > 1 else "32"
precs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["tf32", "bf16"]
for prec in precs:
    for name, r, s, h, c, k in RES:
        cmd = [sys.executable, "tools/run_layer.py", "--h", str(h), "--c", str(c), "--k", str(k), "--r", str(r),
               "--stride", str(s), "--batch", batch, "--prec", prec, "--iters", "2"]
        try:
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=30)
            last = (out.stdout.strip().splitlines() or [out.stderr.strip()[-200:]])[-1]
            print(f"{prec} {name:10s} rc={out.returncode} {last}", flush=True)
        except subprocess.TimeoutExpired:
            print(f"{prec} {name:10s} TIMEOUT", flush=True)
