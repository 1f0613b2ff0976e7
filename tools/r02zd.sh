#!/bin/bash
set -u
WLS="C5 C4" bash tools/variant_sweep.sh r02zd 2 def fr96 fr104 fr112
