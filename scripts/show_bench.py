import json, sys
for f in sys.argv[1:]:
    try: d = json.load(open(f))
    except Exception as e: print(f, e); continue
    r = d['roofline']
    print(f.split('/')[-1], 'ms %.4f' % d['ms_per_step'], 'eager %.4f' % (d.get('eager_ms_per_step') or 0),
          'host %.4f' % d['host_enqueue_ms_per_step'], 'value %.3g' % d['value'],
          'A4 GB/s', r['achieved'] and round(r['achieved']), 'frac', r['frac'] and round(r['frac'], 3),
          'ps_frac', r['ps_apply']['frac'] and round(r['ps_apply']['frac'], 3),
          'roof %.4f' % r['step']['t_roofline_pipelined_ms'], 'stepfrac %.3f' % r['step']['frac_pipelined'],
          'e2e', d['e2e'] and round(d['e2e']['ms_per_step'], 3), 'units', d['config'].get('ps_units'),
          'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
