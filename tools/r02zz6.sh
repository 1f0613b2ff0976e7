#!/bin/bash
set -u
WLS="C5 C4 C3" bash tools/variant_sweep.sh r02zz6 2 def ml0
