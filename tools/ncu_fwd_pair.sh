M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for v in 1 0; do echo "== WF_FWD_PAIR=$v"; WF_FWD_PAIR=$v timeout -s KILL 300 ncu --metrics $M --clock-control none -k regex:wf_block_fwd -s 1 -c 1 --csv python tools/kprof.py 2>/dev/null | grep -v "^==" | tail -3; done
