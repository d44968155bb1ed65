# 4-GPU box: P2P path per pair and the relay probe for owner->helper pairs.
nvidia-smi topo -m > gpurun_out/r2_probe4_topo.txt
nvidia-smi topo -p2p n >> gpurun_out/r2_probe4_topo.txt 2>&1
for pair in "0 2" "0 3" "1 2" "2 0"; do
  echo "== owner/helper $pair" >> gpurun_out/r2_probe4.txt
  timeout 120 ./tools/probe/relay_probe $pair >> gpurun_out/r2_probe4.txt 2>&1
done
