cd /root/repo
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
HXG_PW=1 python -m pytest tests -m gpu -q -x -k "high_order_general or config_parity_protocol or sweep_high_order or specialized" 2>&1 | tail -2
python bench.py --sweep --sweep-reps 2 > gpurun_out/sweep1.json 2>gpurun_out/sweep1.err; tail -2 gpurun_out/sweep1.err
