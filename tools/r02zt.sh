#!/bin/bash
set -u
O=gpurun_out/r02zt; mkdir -p $O
timeout 900 python tools/diag_det.py 1048576 C5 > $O/det_c5.json 2>$O/det_c5.err
timeout 900 python tools/diag_det.py 65536 C4 > $O/det_c4.json 2>$O/det_c4.err
timeout 900 python tools/diag_det.py 16384 C3 > $O/det_c3.json 2>$O/det_c3.err
timeout 900 python tools/diag_det.py 4096 C6 > $O/det_c6.json 2>$O/det_c6.err
