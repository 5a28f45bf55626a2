# ablations of the exact-mode chain kernel at the C2 shapes (see tools/oz_probe.py)
out=gpurun_out/oz_abl.log
: > $out
for a in 0 1 2 3 4 7; do RSVD_OZ_ABLATE=$a python tools/oz_probe.py 50 both 5 >> $out 2>&1; done
RSVD_OZ_ABLATE=0 python tools/oz_probe.py 600 tn 3 >> $out 2>&1
cat $out
