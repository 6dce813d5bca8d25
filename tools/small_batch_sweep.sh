# Member time per schedule and batch (ES_MLP_KERNEL forces a head schedule).
for m in mlp:784,256,10 mlp:784,128,10; do
 for b in 8 16 32 64 128; do
  for k in tmem swapab pair; do
   echo "== $m b=$b kernel=$k"; ES_MLP_KERNEL=$k timeout 120 python tools/time_members.py $m --nb 1048576 --batch $b --steps 5 2>&1 | tail -1
  done
 done
done
