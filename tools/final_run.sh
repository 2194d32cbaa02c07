set -x
mkdir -p gpurun_out/fin
for c in c2 c1 c3 c4 c5; do python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/fin/bench_$c.json 2> gpurun_out/fin/bench_$c.err; done
python bench.py --impl reference --config c2 --steps 20 --warmup 3 > gpurun_out/fin/bench_ref_c2.json 2> gpurun_out/fin/bench_ref_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin/launches_c2.csv python tools/profile_step.py --config c2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin/launches_c3.csv python tools/profile_step.py --config c3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin/launches_c4.csv python tools/profile_subspace.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_bound -c 1 -o gpurun_out/fin/kb_c2 python tools/profile_bound.py --config c2 > gpurun_out/fin/kb_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_bound -c 1 -o gpurun_out/fin/kb_c4 python tools/profile_bound.py --config c4 > gpurun_out/fin/kb_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_bound -c 1 -o gpurun_out/fin/kb_c3 python tools/profile_step.py --config c3 > gpurun_out/fin/kb_c3.log 2>&1
ncu --set full --clock-control none -k regex:k_bound -c 1 -o gpurun_out/fin/kb_c5 python tools/profile_bound.py --config c5 > gpurun_out/fin/kb_c5.log 2>&1
ls gpurun_out/fin
