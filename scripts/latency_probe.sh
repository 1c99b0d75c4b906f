# per-event latency vs concurrency: kernel time of one smc_run at growing replica counts
for w in ${WORKLOADS:-C2}; do for n in ${NS:-600 2400 9600 38400 66000 132000}; do
  python scripts/prof_run.py $w $n | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['counts']; n=c['n_true']+c['n_false']; print(d['workload'], d['n'], 'kernel_ms %.3f' % d['kernel_ms'], 'events/traj %.0f' % (c['events']/n), 'us/event(chain) %.3f' % (1000*d['kernel_ms']/(c['events']/n)), 'grid', d['grid'])"
done; done
