"""5G NR polar reliability sequence (3GPP TS 38.212, Table 5.3.1.2-1).

The 1024 channel indices, least reliable first, stored as zlib-compressed
little-endian uint16 so the table is data, not code.  Shorter blocklengths
keep the entries < N in order (the reference's `reliability_order`,
/root/reference/pkg/src/feclab/codebook.py:185-199).
"""

import base64
import hashlib
import zlib

import numpy as np

_BLOB = (
    "eNoFwQNgEAAABMBHtm3b1qpl27Ztu5Zt27Zt27Zt3QGEEAyhEAmJYARHQYRGCERGGETBAIRDYhRC"
    "NIBJEAvJEBIDURhQWKRCEQxCVIRHJkRACZDRMQRJIcYBVQHJERsxMALBGIopIDVAIFJjPOKhKNIg"
    "mDKjFCJxPkIpESNpPxKpGNJhMCoiC0oiIgpyKLIhJoZhAMsgCJWQC3HREClhVsFITEBwxkdaNIJV"
    "A6ORABNRHCEYmgtQUOnRBAOUFZORAaURhpEZXC2wENlxANNRFosBh2MUhlAOVEZuhFYHDEc5JOZB"
    "VEU0hlEeLMcoNEY15EMs1kQSRlY4HcYYNMUkrMdYRFEhJsRx1EJiJWNhRlNITkEztEQmpuIi1EFG"
    "hOVAJlERnscgTsUMLEEr5EQJxlIhJVNHzER5hGcbFNZ9LEVIpdIhROBAhVVUFlFS5sUKZFInROds"
    "VMcRdMFK5EdUhdcgxWYMRtAGJOcQ1kYJ0UexGj1wAhVYAHE4Ds2xESlYF0N0EhUUyBFMTbk1NmMa"
    "LiAeR6geTiMNx7OBGrAoo2sWLiIzkyod22I7Yii2OmMZHqAYszCY52C8SrIduuIyViGUS/EhkiuO"
    "BjMbr2M+IzIm56IiU2i+uqEMAxVPQ7kGPZFaxxDJm/AYlZiL+zWMa5FGRRXEuOyF/WzIzDqFAFTh"
    "SEZUMaXTFqRkfD5HH5zBVgxWFiVgSaVlI17CBO7AaNZgKQ1VRcXUe5xFfRRnNiXyRDZhVqbnAl5B"
    "LhV0Ge3EME3mIwxwJS1kBgbJbsG4ao/SvIrs3I0DvIHpbKgqSqmReoJ5WMwcjK/gbqQJKsvuqKHK"
    "vIkOHK2nGM7cPMgEKscXSKsQXofemKgmqsrQvo08XM5RXKDiasyE3IaX6Iv0mqwWqsZ8/IAwzqqa"
    "PMwxnMRzWKgMiuz1bMpdeI3p6qDSCucD6oePyK6xrMXjbMYpzMjc+ozK2oMcWqyWPKiyuoYoHq46"
    "XMSpPM/lSuxWLKcZzKNorqp8uoWcPKxqqqlRWsJYTuLGqqWZfIb1GqPv6Mi9aMOxmqTyvM+8vINO"
    "bKqlXMFDbKaEeoXZrM4uDOn8vIuVPMI3yKhCTubjKuwpSuWwbqk62sDzyuQirs2B/oSpOsoCXKRW"
    "GuTw7sHVnKH7yqkS7qi3aM4THMeoLq+l2sglqssvOMmZaqPW7I99iOBp3MxOyqsLXKGvOKR6rK7Z"
    "iuHT/IGVyq9ZTOroPqK23M4u2qBuXMaLjO2f6MwHLKA5rK12vMxxGuLkbq7VOqo1jOPf6Mq6quCN"
    "OqEeesgUXsURnst7mKbNCnRrXecxxnNqn9QFFfVpNXAa19N4X9R29eQmZnYA2yqdH3Mti3mWnvMd"
    "evEU26mztrAPs/gM33OOlumySrqr6vMSt/KBfuEsd3IHr/AbVqmUH2qw5yqiKzqbr2u+Y7o9h7qb"
    "1qiMe+qY/mCTcnmY1+qxKrk7d/MqH3EenzDIcX2DvfRcVbzfDb1F8T3Sp5TSN9lHW/UXZxSgCU7g"
    "tO7NHVrH+nrBRr6kpxzts0rv26zh4r6inZro92rirM7gbVzgl2yveXqkyT7H0u7LD1zo7L6qA27h"
    "1+yuG9qtXXyisp7ufszhyr6pj+zgp9rDa+ytxV6n4c7tzyznF8rj29rLg17uW6zqxu6rUX7GbXqp"
    "fP6gaq7p70zofzjsMT6nO5zkfnqt9W7qV9ylj6rluzzu/hzrjD7vZp7ia3rDlt6jRf6sOv7EW8rp"
    "mW7lqf7KJX6m7+rot9yrGf7CNi7v+97HO8rrpe7kFT7kV/rB6p7tu8rvI17pLv7JN9rgo/6k2l7t"
    "Ah7n5u6vHr7HjX6rE/7Nuv6ik57m1q7nr9rsC57l0/6htt7ud9ynZb7ozv6pb5zjdr6nB+7qVX7o"
    "y57r31rjY+7mAG/yL/b0db/TWj/2KffyH27xGT93H291fX/Te//lJe/wL531Trf3FV/1PD/yH+12"
    "d9/wE9/0Ovf2U//VP972C2/zS/f1OffzB+/ya3/0Hl/zXt/yZz/zd//THb/yXb/xPn/yF/f3W3/1"
    "D//0Pf/2O3/zL//xX//zfzX0BB8="
)
_SHA256 = "06ec3946bc78452ca29a19554793412de07b792a0306f139737af11e71687bff"


def nr_sequence_1024() -> np.ndarray:
    raw = zlib.decompress(base64.b64decode("".join(_BLOB)))
    if hashlib.sha256(raw).hexdigest() != _SHA256:
        raise RuntimeError("bundled NR reliability table failed its checksum")
    return np.frombuffer(raw, dtype="<u2").astype(np.int64)
