#!/bin/bash
# Round-end GPU evidence: parity suite, smoke, default bench line, reference arm,
# config-5 sweep, launch list of the bench command, ncu --set full of the
# dominant kernel per config (+ DRAM traffic per launch for bench.py).
cd "$(dirname "$0")/.."
python -m pytest tests -q -m gpu 2>&1 | tail -2 > gpurun_out/re_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.txt 2>&1
python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/re_bench_ref.json 2> gpurun_out/re_bench_ref.err
[ "${SWEEP:-1}" = 1 ] && python bench.py --sweep > gpurun_out/re_sweep.json 2> gpurun_out/re_sweep.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/re_launches.csv \
    python bench.py --no-suite --no-cpu --steps 2 --warmup 3 --e2e-steps -1 > gpurun_out/re_ncu_bench.log 2>&1
WLS="${WLS:-c2_h1_p5_general:general_v3 c4_hdiv_p7_general:general_v3 c4_l2_p7_general:general_v3}" bash tools/ncu_configs.sh
bash tools/ncu_digest.sh
cat gpurun_out/re_tests.txt gpurun_out/re_smoke.txt
