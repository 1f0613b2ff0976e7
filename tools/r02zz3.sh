#!/bin/bash
set -u
WLS="C5 C4" bash tools/variant_sweep.sh r02zz3 2 def l1p
