cd /root/repo
HXG_PW=1 python tools/pw_diff.py --space H1 --p 7
HXG_PW=1 HXG_LIB=$PWD/paper_1711_00984_b200/_lib_wo0/libhexgram_b200.so python tools/pw_diff.py --space H1 --p 7
for p in 5 6 7; do for s in h1 hcurl; do
  HXG_PW=1 ELEM=1024 bash tools/wl_quick.sh c5_${s}_p${p}_general
  ELEM=1024 bash tools/wl_quick.sh c5_${s}_p${p}_general
done; done
