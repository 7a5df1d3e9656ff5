for ipc in 8 32 64 128; do
  for r in 0 3; do SP_ITEMS_PER_CTA=$ipc python tools/sim_rank_trace.py $r 8 2>&1 | grep '^rank' | sed "s/^/ipc=$ipc /" | cut -c1-60; done
  SP_ITEMS_PER_CTA=$ipc python tools/sim_rank_trace.py 3 8 2>&1 | grep -o "'score_kernel_ms': [0-9.]*"
done
for ipc in 8 32; do SP_ITEMS_PER_CTA=$ipc python tools/sim_rank_trace.py 0 1 2>&1 | grep "^rank" | cut -c1-40; done
