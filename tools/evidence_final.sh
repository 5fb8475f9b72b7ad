#!/bin/bash
# Final evidence of the round (tag $1): tools/evidence_run.sh (bench arms, launch list, ncu --set full per prime at bench size),
# then the lazy mode: ncu of its pipeline, launch list, cross-check against the eager matrix path on fresh seeded surfaces.
tag=$1
tools/evidence_run.sh $tag
for spec in 5:100000 7:100000 11:4000; do
  p=${spec%%:*}; b=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:'k_(caprow|compact_count|compact_scatter|delta_mma|matrix_staged|chain|power_full|fedder)' -s 11 -c 11 -o /tmp/${tag}_lazy_p$p \
      python profiles/run_profile.py --p $p --batch $b --calls 2 --lazy > gpurun_out/${tag}_lazy_p$p.log 2>&1
  python profiles/ncu_summary.py /tmp/${tag}_lazy_p$p.ncu-rep > gpurun_out/${tag}_ncu_lazy_p$p.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/${tag}_launches_lazy.csv python tools/lazy_probe.py > /dev/null 2>&1
{
  python tools/crosscheck.py --p 5 --count 20000000 --seed 6 --lazy
  python tools/crosscheck.py --p 7 --count 10000000 --seed 6 --lazy
  python tools/crosscheck.py --p 3 --count 2000000 --seed 6 --lazy
  python tools/crosscheck.py --p 11 --count 1000000 --block 100000 --seed 6 --lazy
  python tools/crosscheck.py --p 13 --count 200000 --block 50000 --seed 6 --lazy
} > gpurun_out/${tag}_crosscheck_lazy.txt 2>&1
python tools/spectrum.py --p 7 --method lazy --out gpurun_out/${tag}_spectrum_p7_lazy.txt > /dev/null 2>&1
ls -la gpurun_out | tail -20
