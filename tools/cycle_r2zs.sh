# final-tree end-to-end runs of the other BASELINE configs (static_init, frozen-field nu_hat, sweeps to 1e-8 or the cap)
mkdir -p gpurun_out
for spec in "1 400" "2 60" "4 80" "5 10"; do
  set -- $spec
  timeout 600 python tools/run_config.py --config $1 --max-sweeps $2 > gpurun_out/r2zs_run_cfg$1.json 2> gpurun_out/r2zs_run_cfg$1.err; echo cfg $1 rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/r2zs_run_cfg$1.json'))
print('cfg', d['config'], 'sweeps', d['sweeps'], 'converged', d['converged'], 'median sweep ms', round(d['median_sweep_s']*1e3,3), 'DoF/s %.3g' % d['dof_per_s'], 'init_s', round(d['init_s'],2), 'time_s', round(d['time_to_residual_s'],2), 'res ratio %.2e' % (d['history'][-1]/d['history'][0]))"
done
