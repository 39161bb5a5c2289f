"""TEST INFRASTRUCTURE — the CPU oracle for the encrypted-swap hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and the ``--impl reference`` arm) may import this
package, and only as the checker / CPU baseline.  Nothing under
``paper_2411_03357_b200/`` imports it; the product fails loudly when its
CUDA library is missing instead of falling back here.

Two independent restatements of the reference's AES-256-GCM seam
(``specpipe.channel.encrypt_at`` / ``decrypt_at``, channel.py:85-115):

* ``oracle.gcm``  — ctypes over ``gcm_oracle.c`` (FIPS-197 + SP 800-38D,
  bit-serial, no third-party code).  Pinned by the McGrew-Viega TC14 vector
  and by golden vectors generated from the reference itself
  (``tests/golden/gen_golden.py``).
* ``oracle.port`` — the reference's own arithmetic path: the third-party
  ``cryptography`` AESGCM the reference calls (channel.py:23,96,111).  Fast
  (OpenSSL AES-NI); used for large sizes and as the CPU baseline.
"""
