set -x
python bench.py --impl reference > gpurun_out/r02f_bench_c2_reference.json 2> gpurun_out/r02f_ref.err
python bench.py > gpurun_out/r02f_bench_c2.json 2> gpurun_out/r02f_bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02f_c2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-fp64 --no-fp32 --no-c4gemm --no-spmm --no-spectral --graph 0 > gpurun_out/r02f_ncu.log 2>&1
python bench.py --config c1 > gpurun_out/r02f_bench_c1.json 2> gpurun_out/r02f_bench_c1.err
python bench.py --config c5 > gpurun_out/r02f_bench_c5.json 2> gpurun_out/r02f_bench_c5.err
python bench.py --config c5si > gpurun_out/r02f_bench_c5si.json 2> gpurun_out/r02f_bench_c5si.err
python bench.py --config c3 > gpurun_out/r02f_bench_c3.json 2> gpurun_out/r02f_bench_c3.err
python bench.py --config c4 > gpurun_out/r02f_bench_c4.json 2> gpurun_out/r02f_bench_c4.err
ls -la gpurun_out/r02f_*
