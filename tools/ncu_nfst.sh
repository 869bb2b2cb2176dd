#!/bin/bash
out=gpurun_out/ncu5
mkdir -p $out
CID=7 python tools/ozaki_knobs.py "" > $out/knobs.log 2>&1
CID=8 python tools/ozaki_knobs.py "" >> $out/knobs.log 2>&1
CID=7 OP=inv python tools/ozaki_knobs.py "" >> $out/knobs.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:nfst_forward -s 2 -c 1 -o $out/x7_nfst_fwd python tools/profile_step.py X7 > $out/x7.log 2>&1
echo rc=$?
