set -u
WLS="SDF C5" bash tools/variant_sweep.sh r02o 2 def ns
echo done
