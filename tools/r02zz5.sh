#!/bin/bash
set -u
WLS="C5 C3" bash tools/variant_sweep.sh r02zz5 2 def l1p0
