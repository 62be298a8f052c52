cd /root/repo
for w in c5_hdiv_p10_general c5_hdiv_p8_general; do
  python tools/prof_one.py $w --elements 256 --reps 2 > gpurun_out/plain_$w.log 2>&1 || { echo "plain failed $w"; cat gpurun_out/plain_$w.log | tail -5; continue; }
  ncu --set full --clock-control none --import-source on -k regex:general_v2 -s 1 -c 1 -o gpurun_out/prof_$w -f python tools/prof_one.py $w --elements 256 --reps 2 > gpurun_out/ncu_$w.log 2>&1
  tail -1 gpurun_out/ncu_$w.log
done
python bench.py --no-cpu --steps 5 > gpurun_out/bench_dpg.json 2> gpurun_out/bench_dpg.err; tail -2 gpurun_out/bench_dpg.err
