set -u
WLS="C5 C4" bash tools/variant_sweep.sh r02q 2 def ch65536 ch131072 ch262144
echo done
