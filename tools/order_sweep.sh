# per-(dtype, layout, order) time at 2^24 points with the default kernel choices (graph-replayed streams)
mkdir -p gpurun_out
for dt in f64 f32; do for lay in soa aos; do
  if [ $dt = f64 ]; then ORD="0,1,2,3,4,5,6,8,10,12,14,16,20,24,28,32,36"; else ORD="0,1,2,3,4,5,6,8,10,12,14,16"; fi
  echo "$dt $lay $(DTYPE=$dt LAYOUT=$lay timeout 600 python tools/grid_rule.py "$ORD:24" | tail -1)"
done; done
