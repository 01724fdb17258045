import json, sys
for f in sys.argv[1:]:
    d = json.load(open(f))
    print(f)
    for r in d['results']:
        if 'ms' in r:
            o = r['opts']
            print('  %-7s vs=%2d d16=%d seg=%s tile=%5d st=%2s  %8.3f ms  %7.1f GB/s' % (r['variant'], r['vs'], r['d16'], o.get('seg', '-'), r['tile'], o.get('stages', '-'), r['ms'], r['gbs']))
        else:
            print('  ERR', r)
    print(d['summary'])
