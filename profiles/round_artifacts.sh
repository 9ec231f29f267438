#!/bin/bash
# Regenerate the round's bench lines and ncu evidence (run under gpurun;
# outputs land in gpurun_out/, then are copied into profiles/rNN/).
set -u
O=gpurun_out/art
mkdir -p $O
python -m paper_2305_12019_b200.build > /dev/null
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --impl reference > $O/bench_c2_reference_arm.json 2> $O/bench_c2_ref.err
for c in c1 c3 c4; do
  timeout 900 python bench.py --config $c --no-cpu --no-next > $O/bench_$c.json 2> $O/bench_$c.err
done
# launch list of the default command (cold, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-next > $O/ncu_launch.log 2>&1
# one full capture of the persistent kernel (200 iterations in one launch)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_smw_persistent -c 1 \
  -o $O/ncu_persistent_c2 python profiles/run_c2.py 200 > $O/ncu_full.log 2>&1
ncu -i $O/ncu_persistent_c2.ncu-rep --page raw --csv > $O/ncu_persistent_c2_raw.csv 2>/dev/null
python profiles/ncu_summary.py $O/ncu_persistent_c2_raw.csv > $O/ncu_persistent_c2_summary.csv
# per-phase timing of the persistent kernel (CTA clock stamps), c2 and c1
GDWD_PK_TIMING=1 timeout 300 python profiles/run_c2.py 100 > $O/persistent_phase_timing.txt 2>&1
# one full capture of the feature-blocked sparse Z~^T w kernel (config 4)
timeout 900 ncu --set full --clock-control none -k regex:sp_ztmv_fb_kernel -s 2 -c 1 -o $O/ncu_c4_sp_ztmv_fb \
  python bench.py --config c4 --no-cpu --no-next --no-e2e --steps 3 --warmup 3 > $O/ncu_fb.log 2>&1
ncu -i $O/ncu_c4_sp_ztmv_fb.ncu-rep --page raw --csv > $O/ncu_c4_sp_ztmv_fb_raw.csv 2>/dev/null
python profiles/ncu_summary.py $O/ncu_c4_sp_ztmv_fb_raw.csv > $O/ncu_c4_sp_ztmv_fb.csv
timeout 1500 python bench.py --config c5 --no-cpu --no-next > $O/bench_c5.json 2> $O/bench_c5.err
echo done
