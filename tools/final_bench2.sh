set -x
python bench.py --config c5 > gpurun_out/r02g_bench_c5.json 2> gpurun_out/r02g_bench_c5.err
python bench.py --config c5si > gpurun_out/r02g_bench_c5si.json 2> gpurun_out/r02g_bench_c5si.err
python bench.py --config c3 > gpurun_out/r02g_bench_c3.json 2> gpurun_out/r02g_bench_c3.err
python bench.py --config c4 > gpurun_out/r02g_bench_c4.json 2> gpurun_out/r02g_bench_c4.err
ls -la gpurun_out/r02g_*
