#!/bin/bash
set -u
WLS="C5 C4" bash tools/variant_sweep.sh r02zz8 2 def tb0
