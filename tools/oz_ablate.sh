python tools/oz_probe.py 50 both 5 > gpurun_out/r02_oz_abl.log 2>&1; python tools/oz_probe.py 600 tn 3 >> gpurun_out/r02_oz_abl.log 2>&1
for a in 1 2 3 4; do echo "ablate $a" >> gpurun_out/r02_oz_abl.log; RSVD_OZ_ABLATE=$a python tools/oz_probe.py 50 both 5 >> gpurun_out/r02_oz_abl.log 2>&1; done
timeout 300 python -m pytest tests/test_gpu_oz.py -x -q -s > gpurun_out/r02_oz_test.log 2>&1
