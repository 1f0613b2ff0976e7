set -u
WLS="SDF" bash tools/variant_sweep.sh r02s 2 def sxo
echo done
