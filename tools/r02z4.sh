#!/bin/bash
set -u
WLS="C5 C4 C3" bash tools/variant_sweep.sh r02z4 2 def lv0
WLS="SDF" bash tools/variant_sweep.sh r02z4 2 def lv0
