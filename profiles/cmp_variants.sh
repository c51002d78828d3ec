for v in paper_1805_06572_b200/lib/libfastfca_b200.so paper_1805_06572_b200/lib/var/*.so; do
  FFCA_LIBRARY=$v python bench.py --steps 5 --streams 1 > /tmp/b.json 2> /tmp/b.err || tail -3 /tmp/b.err
  python -c "import json; d=json.load(open('/tmp/b.json')); r=d['roofline']; print('$v'.split('/')[-1], round(d['value']/1e9,2), round(d['ms_per_step'],2), r['kernel_ms_avg'], r['last_pass_with_images_ms'], d['clocks']['sm_mhz'])"
done
