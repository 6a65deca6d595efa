timeout 300 python tools/iter_profile.py c4 3e-3 0.8 --bucket 2000 2>&1 | grep -v "^loop"
echo "== c2 no PDL"; KRONRED_NO_PDL=1 timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep "after pick\|^sum\|total device\|pick start"
echo "== c2"; timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep "after pick\|^sum\|total device\|pick start"
