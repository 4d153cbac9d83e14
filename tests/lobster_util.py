"""Test helpers: LOBSTER message/orderbook pairs written the way the reference's
write_lobster does (data/lobster.hpp:195-236: %d.%09d times, type = kind + 1,
price * units_per_tick, orderbook rows from replaying the messages through a
book, sentinel-padded to `depth` levels), and the malformed-input cases the
reference's loader rejects (test_data.cpp:84-113 and the other checks of
lobster.hpp:119-190)."""
from oracle.oracle import OBook


def write_lobster(o, msgs, msg_path, book_path, upt=100, depth=5):
    book = OBook(o, 1 << 18)
    with open(msg_path, "w") as mf, open(book_path, "w") as bf:
        for m in msgs:
            t = int(m["time"])
            mf.write(f"{t // 1000000000}.{t % 1000000000:09d},{int(m['kind']) + 1},{int(m['order_id'])},"
                     f"{int(m['quantity'])},{int(m['price']) * upt},{1 if int(m['side']) == 0 else -1}\n")
            book.process(m)
            bids, asks = book.l2(depth)
            cols = []
            for lv in range(depth):
                cols += [f"{asks[lv][0] * upt},{asks[lv][1]}" if lv < len(asks) else "9999999999,0"]
                cols += [f"{bids[lv][0] * upt},{bids[lv][1]}" if lv < len(bids) else "-9999999999,0"]
            bf.write(",".join(cols) + "\n")


# (name, message file text, orderbook file text, units_per_tick, sample_every)
MALFORMED = [
    ("fewer_book_rows", "1.0,1,1,1,100,1\n2.0,1,2,1,100,1\n", "100,1,90,1\n", 1, 1),
    ("fewer_msg_rows", "1.0,1,1,1,100,1\n", "100,1,90,1\n100,1,90,1\n", 1, 1),
    ("bad_id", "1.0,1,1,1,100,1\n2.0,1,xyz,1,100,1\n", "100,1,90,1\n100,1,90,1\n", 1, 1),
    ("non_monotone", "2.0,1,1,1,100,1\n1.0,1,2,1,100,1\n", "100,1,90,1\n100,1,90,1\n", 1, 1),
    ("negative_first_time", "-5.0,1,1,1,100,1\n", "100,1,90,1\n", 1, 1),
    ("five_fields", "1.0,1,1,1,100\n", "100,1,90,1\n", 1, 1),
    ("empty_fraction", "1.,1,1,1,100,1\n", "100,1,90,1\n", 1, 1),
    ("bad_fraction", "1.2x,1,1,1,100,1\n", "100,1,90,1\n", 1, 1),
    ("bad_seconds", "a.5,1,1,1,100,1\n", "100,1,90,1\n", 1, 1),
    ("unknown_type", "1.0,9,1,1,100,1\n", "100,1,90,1\n", 1, 1),
    ("bad_type", "1.0,+1,1,1,100,1\n", "100,1,90,1\n", 1, 1),
    ("negative_size", "1.0,1,1,-3,100,1\n", "100,1,90,1\n", 1, 1),
    ("bad_size", "1.0,1,1,3 ,100,1\n", "100,1,90,1\n", 1, 1),
    ("price_tick", "1.0,1,1,3,105,1\n", "100,1,90,1\n", 10, 1),
    ("bad_price", "1.0,1,1,3,1e5,1\n", "100,1,90,1\n", 1, 1),
    ("direction", "1.0,1,1,3,100,0\n", "100,1,90,1\n", 1, 1),
    ("bad_direction", "1.0,1,1,3,100,x\n", "100,1,90,1\n", 1, 1),
    ("book_columns", "1.0,1,1,3,100,1\n", "100,1,90\n", 1, 1),
    ("book_field", "1.0,1,1,3,100,1\n", "100,1,90,q\n", 1, 1),
    ("book_tick", "1.0,1,1,3,100,1\n", "105,1,90,1\n", 10, 1),
    ("book_tick_bid", "1.0,1,1,3,100,1\n", "100,1,95,1\n", 10, 1),
    ("overflow_id", "1.0,1,99999999999999999999,3,100,1\n", "100,1,90,1\n", 1, 1),
    ("second_row_book", "1.0,1,1,3,100,1\n2.0,1,2,3,100,1\n", "100,1,90,1\nbad\n", 1, 2),
    ("first_error_wins", "1.0,1,1,3,100,1\n0.5,1,x,3,100,1\n0.4,9,1,3,100,1\n",
     "100,1,90,1\n100,1,90,1\n100,1,90,1\n", 1, 1),
]

# accepted inputs with edge cases: blank / CRLF lines, unsampled malformed book rows,
# trailing blank book rows, a state keyed one past the last message (dropped)
ACCEPTED = [
    ("kat", "34200.000123, 1, 42, 10, 3148000, 1\n34200.000124, 7, 0, 0, 3148000, -1\n",
     "3149000,5,3148000,10\n3149000,5,3148000,10\n", 100, 1),
    ("crlf_and_blank", "1.5,1,1,3,100,1\r\n\n\r\n2.25,2,1,1,100,1\r\n3,4,1,1,100,1",
     "100,1,90,1\r\n100,2,90,2\r\nnot,a,book,row\n\n\n", 1, 2),
    ("unsampled_bad_book", "1.0,1,1,3,100,1\n2.0,1,2,3,100,-1\n3.0,3,1,0,100,1\n",
     "x\n100,1,90,1,110,2,80,3\ny\n", 1, 2),
    ("sentinels", "1.000000001,1,1,3,100,1\n1.0000000019,5,0,1,100,-1\n",
     "9999999999,0,-9999999999,0\n200,0,90,0,110,4,0,7\n", 1, 1),
    ("no_messages", "\n\n", "", 1, 1),
]
