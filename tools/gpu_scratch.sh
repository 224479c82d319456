O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"radix_scatter|radix_hist|mp_diff_keys" -s 20 -c 3 -o $O/prof_tc_sort python tools/phase_report.py --workload tc --kernels > $O/ncu_tc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"wcoj_kernel<0, 2>" -s 100 -c 2 -o $O/prof_doop_gen python tools/phase_report.py --workload doop --kernels > $O/ncu_doopg.log 2>&1
exit 0
