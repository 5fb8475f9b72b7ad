#!/bin/bash
# session-3 evidence: full GPU tests, sanitizer on the lazy path, F_7 spectrum search lazy vs matrix, ncu of the lazy pipeline
python -m pytest tests -m gpu -x -q > gpurun_out/s3c_gputests.log 2>&1; echo "exit $?" >> gpurun_out/s3c_gputests.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py 3,5,7,11 > gpurun_out/r2h_sanitizer_memcheck.txt 2>&1
python tools/spectrum.py --p 7 --method lazy --out gpurun_out/r2h_spectrum_p7_lazy.txt > gpurun_out/r2h_spectrum_p7_lazy.log 2>&1
python tools/spectrum.py --p 5 --method lazy --out gpurun_out/r2h_spectrum_p5_lazy.txt > gpurun_out/r2h_spectrum_p5_lazy.log 2>&1
for spec in 5:100000 7:100000 11:4000; do
  p=${spec%%:*}; b=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:'k_(caprow|delta_mma|matrix_staged|chain|power_full|fedder|compact)' -s 9 -c 9 -o /tmp/r2h_lazy_p$p \
      python profiles/run_profile.py --p $p --batch $b --calls 2 --lazy > gpurun_out/r2h_lazy_p$p.log 2>&1
  python profiles/ncu_summary.py /tmp/r2h_lazy_p$p.ncu-rep > gpurun_out/r2h_ncu_lazy_p$p.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2h_launches_lazy.csv python tools/lazy_probe.py > /dev/null 2>&1
ls -la gpurun_out | tail -12
