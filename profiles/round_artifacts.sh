#!/bin/bash
# Regenerate the round's bench lines and ncu evidence (run under gpurun;
# outputs land in gpurun_out/art, then are copied into profiles/rNN/).
set -u
O=gpurun_out/art
mkdir -p $O
python -m paper_2305_12019_b200.build > /dev/null
# the driver's command
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_c2_reference_arm.json 2> $O/bench_c2_ref.err
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-next --no-anchor --kkt-iters 0 > $O/bench_c2_k200.json 2> $O/bench_c2_k200.err
for c in c1 c3 c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-next --no-anchor > $O/bench_$c.json 2> $O/bench_$c.err
done
# end-to-end split and the device timeline of the pipelined upload (copy / Gram rows / factor rows / G^-1 terms)
GDWD_SETUP_TIMING=1 timeout 300 python profiles/e2e_probe.py c2 20 4 > $O/upload_timeline_c2.txt 2>&1
# launch list of the default command (cold, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-next --no-anchor --kkt-iters 0 > $O/ncu_launch.log 2>&1
# one full capture of the persistent kernel (200 iterations in one launch)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_smw_persistent -c 1 \
  -o $O/ncu_persistent_c2 python profiles/run_c2.py 200 > $O/ncu_full.log 2>&1
ncu -i $O/ncu_persistent_c2.ncu-rep --page raw --csv > $O/ncu_persistent_c2_raw.csv 2>/dev/null
python profiles/ncu_summary.py $O/ncu_persistent_c2_raw.csv > $O/ncu_persistent_c2_summary.csv
# one full capture of the DMMA Gram kernel (c2 Z^T Z)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_tile_kernel -s 1 -c 1 \
  -o $O/ncu_gram_tile python profiles/run_gram_c2.py > $O/ncu_gram.log 2>&1
ncu -i $O/ncu_gram_tile.ncu-rep --page raw --csv > $O/ncu_gram_tile_raw.csv 2>/dev/null
python profiles/ncu_summary.py $O/ncu_gram_tile_raw.csv > $O/ncu_gram_tile_summary.csv
# per-phase timing of the persistent kernel (CTA clock stamps)
GDWD_PK_TIMING=1 timeout 300 python profiles/run_c2.py 100 > $O/persistent_phase_timing.txt 2>&1
# sparse kernels of config 4
timeout 900 ncu --set full --clock-control none -k regex:"sp_ztmv_fb_kernel|sp_zmv_sb_kernel" -s 4 -c 2 -o $O/ncu_c4_sparse \
  python bench.py --config c4 --no-cpu --no-next --no-e2e --no-anchor --kkt-iters 0 --steps 3 --warmup 3 > $O/ncu_c4.log 2>&1
ncu -i $O/ncu_c4_sparse.ncu-rep --page raw --csv > $O/ncu_c4_sparse_raw.csv 2>/dev/null
python profiles/ncu_summary.py $O/ncu_c4_sparse_raw.csv > $O/ncu_c4_sparse_summary.csv
# fused tail of config 3
timeout 900 ncu --set full --clock-control none -k regex:zft_kernel -s 2 -c 1 -o $O/ncu_c3_zft \
  python bench.py --config c3 --no-cpu --no-next --no-e2e --no-anchor --kkt-iters 0 --steps 3 --warmup 3 > $O/ncu_c3.log 2>&1
ncu -i $O/ncu_c3_zft.ncu-rep --page raw --csv > $O/ncu_c3_zft_raw.csv 2>/dev/null
python profiles/ncu_summary.py $O/ncu_c3_zft_raw.csv > $O/ncu_c3_zft_summary.csv
timeout 1500 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu --no-next > $O/bench_c5.json 2> $O/bench_c5.err
rm -f $O/*.ncu-rep
echo done
