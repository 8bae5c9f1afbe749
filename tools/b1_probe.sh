for mode in auto im2col pixn halo; do
  for sp in 0 1 2 4 8 16; do
    echo "=== mode=$mode split=$sp"
    timeout 120 python tools/layer_times.py vgg16 tf32 1 --mode $mode --split $sp 2>&1 | grep -v '^tilekit\|^layer'
  done
done
