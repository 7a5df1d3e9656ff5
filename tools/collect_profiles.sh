# Round-2 measurement set (one B200): bench line + reference arm, every
# BASELINE config, the simulated strong scaling, the fold at scale, launch
# lists of the c5 step (both scoring modes) and of the small configs, and
# full ncu captures of the small-search kernel.  Outputs in gpurun_out/.
set -x
python bench.py > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
python bench.py --impl reference > gpurun_out/r2_bench_c5_reference.json 2> gpurun_out/r2_bench_ref.err
bash tools/all_configs.sh gpurun_out/r2_configs.jsonl 2> gpurun_out/configs.err
python tools/shard_sim.py 5 > gpurun_out/r2_shard_sim_c5.txt 2>&1
python tools/shard_sim.py 5 --host-exchange > gpurun_out/r2_shard_sim_c5_host_exchange.txt 2>&1
python tools/fold_scale.py --layers 1000 100000 700000 --out gpurun_out/r2_fold_scale.json > gpurun_out/fold_scale.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fold10m.csv python tools/fold_scale.py --layers 700000 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5_walk.csv python tools/ncu_target.py c5 walk 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5_skip.csv python tools/ncu_target.py c5 skip 2 > /dev/null 2>&1
for w in c1 c3 c4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_$w.csv python tools/ncu_target.py $w skip 3 > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:"k_search_small|k_fold_small|k_fill" --launch-skip 6 -c 3 -o gpurun_out/r2_small_c4 python tools/ncu_target.py c4 skip 4 > /dev/null 2>&1
