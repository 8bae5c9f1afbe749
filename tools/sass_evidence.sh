#!/bin/sh
# Per-kernel SASS evidence for profiles/: counts of the tcgen05 / TMA / exact
# FP32 mnemonics in the built library, plus the full SASS of the dominant
# tensor-core kernel.   sh tools/sass_evidence.sh r01
set -e
R=${1:-r01}
cd "$(dirname "$0")/.."
cuobjdump -sass paper_1904_05347_b200/libtilekit_b200.so > /tmp/tk_all.sass
python3 - "$R" <<'PY'
import collections, re, subprocess, sys
txt = open("/tmp/tk_all.sass").read()
out = []
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n", 1)[0].strip()
    c = collections.Counter()
    for k in re.findall(r"\b(UTC\w*MMA\w*|UTMALDG(?:\.\w+)*|UTMASTG\w*|UBLKCP\w*|LDTM\w*|STTM\w*|"
                        r"HMMA\w*|FFMA|FMUL|FADD|LDGSTS\w*|SYNCS\.\w+)", f):
        c[k if k.startswith("SYNCS") else (k if k.startswith("UTMALDG") else k.split(".")[0])] += 1
    out.append((name, c))
dem = subprocess.run(["c++filt"], input="\n".join(n for n, _ in out), capture_output=True,
                     text=True).stdout.split("\n")
with open(f"profiles/{sys.argv[1]}_sass_mnemonics.txt", "w") as fo:
    fo.write("# cuobjdump -sass paper_1904_05347_b200/libtilekit_b200.so: per-kernel counts of the\n"
             "# instructions that prove the tcgen05/TMA (UTC*MMA, UTMALDG/UTMASTG, LDTM) and\n"
             "# exact-FP32 (FMUL+FADD, no FFMA) paths.  Regenerate: sh tools/sass_evidence.sh\n\n")
    for (n, c), d in zip(out, dem):
        if c:
            fo.write(d[:160] + "\n    " + ", ".join(f"{k}={v}" for k, v in sorted(c.items())) + "\n")
PY
# Full SASS of the pixN TF32 CTA-pair kernel (58% of the VGG16 step).
awk '/Function : .*tc_gemm_kernelILi1ELi2ELb1E/{f=1; print; next} f&&/Function : /{f=0} f' \
  /tmp/tk_all.sass > "profiles/${R}_sass_tc_gemm_pixN_cg2_tf32.txt"
wc -l profiles/${R}_sass_*.txt
