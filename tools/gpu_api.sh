# SSSP engine width A/B on the grid (degree 4) and the band (degree 256)
export PYTHONPATH=.
for nw in 4 2 1 8 4; do
  PBH_SSSP_NW=$nw timeout 300 python tools/probe_sssp.py exact grid 2048 2 2>&1 | tail -1 | sed "s/^/nw=$nw /" | cut -c1-200
  PBH_SSSP_NW=$nw timeout 300 python tools/probe_sssp.py exact band 18 1 2>&1 | tail -1 | sed "s/^/nw=$nw /" | cut -c1-200
done
