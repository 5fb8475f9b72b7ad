#!/bin/bash
# One evidence run on the GPU box (gpurun): bench lines of both arms, the ncu launch list of the bench command, and one
# `ncu --set full` capture per prime AT THE BENCHMARK'S LAUNCH SIZE, reduced on the box to text (the reports themselves exceed
# what gpurun copies back).  Afterwards, here: python profiles/collect.py TAG
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'tools/evidence_run.sh r2a'
tag=$1
K='k_(delta_mma|matrix_staged|chain|power_full|fedder|delta_box|delta_prep)'
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${tag}_ref.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 1 --cpu-seconds 1 > /dev/null 2>&1
for spec in 5:100000 7:100000 11:4000; do
  p=${spec%%:*}; b=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s 7 -c 7 -o /tmp/${tag}_full_p$p \
      python profiles/run_profile.py --p $p --batch $b --calls 2 > gpurun_out/${tag}_full_p$p.log 2>&1
  python profiles/ncu_summary.py /tmp/${tag}_full_p$p.ncu-rep > gpurun_out/${tag}_full_p$p.summary.txt
  python profiles/ncu_lines.py /tmp/${tag}_full_p$p.ncu-rep 40 > gpurun_out/${tag}_full_p$p.lines.txt
  ncu -i /tmp/${tag}_full_p$p.ncu-rep --page raw --csv > gpurun_out/${tag}_full_p$p.raw.csv 2>/dev/null
done
ls -la gpurun_out | tail -15
