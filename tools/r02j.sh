set -u
bash tools/variant_sweep.sh r02j 2 r1 def a0 b0 c0 d0
echo done
