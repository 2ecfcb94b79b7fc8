cp paper_2008_01938_b200/_lib/libpipedp_cuda.so /tmp/orig.so
for v in orig ap128 ap192; do
  if [ $v != orig ]; then cp tools/libexp_$v.so paper_2008_01938_b200/_lib/libpipedp_cuda.so; fi
  echo $v; PIPEDP_SDP_CHUNKED=0 python tools/cluster_probe.py 20 | tail -1
done
