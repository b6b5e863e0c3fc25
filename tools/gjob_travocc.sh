bash tools/gjob_ab.sh "C2 C4" default ab/libpxg_trav8.so ab/libpxg_trav6.so
