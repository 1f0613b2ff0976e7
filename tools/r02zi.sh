#!/bin/bash
set -u
WLS="SDF" bash tools/variant_sweep.sh r02zi 3 def st64 st128
