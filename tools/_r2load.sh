# Measured serving of C3 shard 0 of 8 at 1x / 4x / 16x the reference's
# offered load (arrival and think times compressed): queueing gives the
# pre-loader its read-buffer head start.
set -x
mkdir -p gpurun_out
for L in 1 4 16; do
  timeout 1200 python -m paper_2403_19708_b200.serve --config c3 --of 8 --shard 0 --dram-gb 96 --load $L --json gpurun_out/r2al_serve_load$L.json > gpurun_out/r2al_serve_load$L.log 2>&1
  echo "load $L rc=$?"
done
